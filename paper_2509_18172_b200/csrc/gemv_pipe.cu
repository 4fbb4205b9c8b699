// gemv_pipe.cu -- SBVR GEMV at batch 1 (§4.4) as a persistent, warp-specialised
// kernel: the AND+popcount inner products of gemv_mma.cu (bit-sliced u8 mma.sync, see there) fed by
// a CTA-wide TMA ring and scheduled dynamically, with a deterministic split-K combine.
//
// Why (profiles/r01_phase_step.json): with static per-warp ranges the 4 GEMV launches of a decode
// step lost ~40% of their span to stragglers -- late-starting SMs (the previous kernel's tail) got
// their first bytes last and finished last, and owner CTAs waited for late publishers.  Here every
// CTA (one per SM) runs three roles:
//   producer warp  : takes work items (a static prefix before griddepcontrol.wait, then tickets from
//                    a global atomic counter), one cp.async.bulk per item into an S-stage ring
//                    (mbarrier complete_tx), L2 evict-first (weights are streamed once).
//   16 consumer warps: per stage, warp w computes tile pair (w & 3) of unit (w >> 2) of the item
//                    (the tile compute and epilogue of gemv_mma.cu), quad-reduces its rows and hands
//                    them to the flush warp through a shared-memory partial ring.
//   flush warp     : sums the 4 unit contributions of every row in unit order; an item that does not
//                    cover the whole row block stores its partial in a global slot; the item holding
//                    the row block's last chunk (it is ticketed after all the others) pulls the other
//                    chunks' partials (sentinel-checked, no flags or atomics), adds them in chunk order
//                    (deterministic), writes y and re-arms the slots.
// Work item = (row block rb of 128 rows, chunk of UPS consecutive groups): the UPS unit records of
// the item are contiguous in HBM (sbvr.h), so one bulk copy moves the whole item.  Every wait points
// to an item with a smaller index and each CTA processes its items in increasing index order, so the
// persistent grid (<= one CTA per SM, all co-resident) cannot deadlock.
#include <cstdlib>

#include "sbvr_internal.cuh"

namespace sbvr {
namespace {

constexpr int kCons = 16;                        // consumer warps
constexpr int kProdWarp = kCons, kFlushWarp = kCons + 1, kRedWarp = kCons + 2;
constexpr int kWarps = kCons + 3;
constexpr int kPipeThreads = kWarps * 32;
constexpr int kRQ = 4;                           // reduction queue depth (flush warp -> reducer warp)
constexpr int kUPS = 4;                          // units (groups) per item
constexpr int kPS = 8;                           // partial ring depth
constexpr int kMaxStages = 6;
constexpr unsigned int kSent = 0xFFFFFFFFu;      // empty partial slot (a NaN arithmetic never produces)

struct PipeParams {
  const uint8_t* units;
  const float* ratio_pow;     // [n_ratio][K]
  const uint32_t* xplanes;    // [NG][l][4]
  const float* xscales;       // [NG]
  float* Y;                   // [M]
  int32_t* P;                 // debug partials [M][NG][K][l] (DEBUG only)
  float* part;                // [n_rb][nc][128] partial slots, kSent when empty
  unsigned int* ticket;       // dynamic work counter (0xFFFFFFFF at rest)
  int M, N, l, n_ratio;
  int n_full, tail_rows, n_rb, NG, nc, n_items;
  int S;                      // stages
  int stage_bytes;
  int x_bytes;                // shared-memory bytes of the staged activation planes
  int one;                    // = 1 (runtime, keeps the magic-number IMAD on the FMA pipe)
  unsigned long long* ts;     // diagnostics (env SBVR_TS_PTR): [CTA][warp][8]
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_ef(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const float* ptr) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t bslice(uint32_t X, int s) {
  // byte b of the result = bit (8b + s) of X placed at bit (7 - s) of byte b
  const int sh = 7 - 2 * s;
  const uint32_t y = sh >= 0 ? (X << sh) : __umulhi(X, 1u << (32 + sh));
  return y & (0x01010101u << (7 - s));
}
__device__ __forceinline__ void mma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1, int c0, int c1, int c2, int c3) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}
__device__ __forceinline__ int imad(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

#define PTS(slot, val) do { if (p.ts && lane == 0) p.ts[((size_t)blockIdx.x * kWarps + wib) * 8 + (slot)] = (val); } while (0)

template <int K, bool DEBUG>
__global__ void __launch_bounds__(kPipeThreads, 1) gemv_pipe_kernel(PipeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], pfull_bar[kPS], pempty_bar[kPS];
  __shared__ int s_hdr[kMaxStages];      // item of each stage (-1 = no more work)
  __shared__ int s_phdr[kPS];            // item of each partial slot
  __shared__ float s_rat[64];
  __shared__ uint64_t rfull_bar[kRQ], rempty_bar[kRQ];
  __shared__ int s_rrb[kRQ];             // row block of each queued reduction (-1 = done)
  __shared__ float s_rval[kRQ][128];     // the last chunk's own partial
  // dynamic smem: [stages][partial ring: kPS x kCons x 32 floats][x planes NG*l*4 u32][x scales NG]
  uint8_t* stages = smem;
  float* s_part = reinterpret_cast<float*>(smem + (size_t)p.S * p.stage_bytes);
  uint32_t* s_xp = reinterpret_cast<uint32_t*>(s_part + kPS * kCons * 32);
  float* s_xs = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(s_xp) + p.x_bytes);

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  PTS(0, gtime());
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(full_bar + s, 1);
      mbar_init(empty_bar + s, kCons);
    }
    for (int s = 0; s < kPS; ++s) {
      mbar_init(pfull_bar + s, kCons);
      mbar_init(pempty_bar + s, 1);
    }
    for (int s = 0; s < kRQ; ++s) {
      mbar_init(rfull_bar + s, 1);
      mbar_init(rempty_bar + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < p.n_ratio; i += blockDim.x) s_rat[i] = K >= 2 ? p.ratio_pow[i * K + 1] : 0.f;
  __syncthreads();

  const int G = gridDim.x;
  // ---------------------------------------------------------------- producer
  if (wib == kProdWarp) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      auto load = [&](int slot, int v) {
        s_hdr[slot] = v;
        if (v < 0) {
          mbar_arrive(full_bar + slot);
          return;
        }
        const int rb = v / p.nc, c = v - rb * p.nc;
        const int g0 = c * kUPS, ng = min(kUPS, p.NG - g0);
        const int R = rb < p.n_full ? 128 : p.tail_rows;
        const size_t ub = (size_t)R * (16 * K + 5);
        const uint8_t* src = rb < p.n_full ? p.units + ((size_t)rb * p.NG + g0) * ub
                                           : p.units + (size_t)p.n_full * p.NG * (128 * (16 * K + 5)) + (size_t)g0 * ub;
        mbar_expect_tx(full_bar + slot, (uint32_t)(ng * ub));
        bulk_g2s_ef(stages + (size_t)slot * p.stage_bytes, src, (uint32_t)(ng * ub), full_bar + slot, pol);
      };
      // static prefix: weights are immutable, so they stream before the previous kernel completes
      int it = 0;
      // (contiguous blocks: a row block's chunks land in at most a few neighbouring CTAs and the
      // reductions -- one per row block, done by the holder of its last chunk -- spread evenly)
      const int pre = min(p.n_items, p.S * G);           // prefix items, split in balanced contiguous blocks
      const int pb0 = (int)((long)blockIdx.x * pre / G), pb1 = (int)((long)(blockIdx.x + 1) * pre / G);
      for (; it < pb1 - pb0; ++it) load(it, pb0 + it);
      asm volatile("griddepcontrol.wait;" ::: "memory");   // the ticket counter was reset by the previous launch
      if (DEBUG) {                                        // no workspace: the static schedule only
        for (;; ++it) {
          const int slot = it % p.S;
          if (it >= p.S) mbar_wait(empty_bar + slot, ((it / p.S) - 1) & 1);
          const int v = p.S * G + (it - (pb1 - pb0)) * G + blockIdx.x;   // static round robin after the prefix
          load(slot, v < p.n_items ? v : -1);
          if (v >= p.n_items) break;
        }
        return;
      }
      const unsigned int total = (unsigned int)(G + max(0, p.n_items - pre));
      unsigned long long t_empty = 0, t_ticket = 0;
      // the next ticket is drawn as soon as the previous item is issued, so its round trip overlaps the
      // wait for a free stage (0-based ticket; the counter rests at 0xFFFFFFFF)
      unsigned int t_next = atomicAdd(p.ticket, 1u) + 1u;
      for (;; ++it) {
        const int slot = it % p.S;
        unsigned long long ta = p.ts ? gtime() : 0;
        if (it >= p.S) mbar_wait(empty_bar + slot, ((it / p.S) - 1) & 1);
        unsigned long long tb = p.ts ? gtime() : 0;
        const unsigned int t = t_next;
        if (p.ts) {
          const unsigned long long tc = gtime();
          t_empty += tb - ta;
          t_ticket += tc - tb;
          p.ts[((size_t)blockIdx.x * kWarps + wib) * 8 + 5] = t_empty;
          p.ts[((size_t)blockIdx.x * kWarps + wib) * 8 + 6] = t_ticket;
          p.ts[((size_t)blockIdx.x * kWarps + wib) * 8 + 7] = it + 1;
        }
        const int v = pre + (int)t;
        if (v < p.n_items) {
          load(slot, v);
          t_next = atomicAdd(p.ticket, 1u) + 1u;
          continue;
        }
        if (t == total - 1) atomicExch(p.ticket, 0xFFFFFFFFu);  // last draw of this launch: re-arm
        load(slot, -1);
        break;
      }
    }
    PTS(3, gtime());
    return;
  }

  // ---------------------------------------------------------------- flush warp
  if (wib == kFlushWarp) {
    if (DEBUG) return;
    asm volatile("griddepcontrol.wait;" ::: "memory");     // y and the partial slots are ours from here
    int nred = 0;
    for (int k = 0;; ++k) {
      const int ps = k % kPS;
      mbar_wait(pfull_bar + ps, (k / kPS) & 1);
      const int v = s_phdr[ps];
      if (v < 0) break;
      const int rb = v / p.nc, c = v - rb * p.nc;
      const int R = rb < p.n_full ? 128 : p.tail_rows;
      float mine[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {                      // row q*32 + lane = tile pair q, row-in-pair lane
        float s = 0.f;
#pragma unroll
        for (int u = 0; u < kUPS; ++u) s += s_part[((size_t)ps * kCons + u * 4 + q) * 32 + lane];
        mine[q] = s;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(pempty_bar + ps);
      float* yrow = p.Y + (size_t)rb * 128;
      if (p.nc > 1 && c == p.nc - 1) {                 // the row block's last chunk: queue its reduction
        const int rq = nred % kRQ;
        if (nred >= kRQ) mbar_wait(rempty_bar + rq, ((nred / kRQ) - 1) & 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) s_rval[rq][q * 32 + lane] = mine[q];
        if (lane == 0) s_rrb[rq] = rb;
        __syncwarp();
        if (lane == 0) mbar_arrive(rfull_bar + rq);
        ++nred;
        continue;
      }
      if (p.nc == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q * 32 + lane < R) yrow[q * 32 + lane] = mine[q];
        continue;
      }
      float* slots = p.part + (size_t)rb * p.nc * 128;
#pragma unroll
      for (int q = 0; q < 4; ++q) __stcg(slots + (size_t)c * 128 + q * 32 + lane, mine[q]);
    }
    {                                                    // tell the reducer warp we are done
      const int rq = nred % kRQ;
      if (nred >= kRQ) mbar_wait(rempty_bar + rq, ((nred / kRQ) - 1) & 1);
      if (lane == 0) {
        s_rrb[rq] = -1;
        mbar_arrive(rfull_bar + rq);
      }
    }
    PTS(3, gtime());
    return;
  }

  // ---------------------------------------------------------------- reducer warp
  if (wib == kRedWarp) {
    if (DEBUG) return;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int k = 0;; ++k) {
      const int rq = k % kRQ;
      mbar_wait(rfull_bar + rq, (k / kRQ) & 1);
      const int rb = s_rrb[rq];
      if (rb < 0) break;
      float mine[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) mine[q] = s_rval[rq][q * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(rempty_bar + rq);
      const int R = rb < p.n_full ? 128 : p.tail_rows;
      float* yrow = p.Y + (size_t)rb * 128;
      float* slots = p.part + (size_t)rb * p.nc * 128;
      // pull the other chunks' partials in chunk order, sum, write y, re-arm
      const unsigned long long tr0 = p.ts ? gtime() : 0;
      float tot[4] = {0.f, 0.f, 0.f, 0.f};
      constexpr int kB = 8;
      for (int c0 = 0; c0 < p.nc - 1; c0 += kB) {
        uint32_t vals[kB][4];
        // reload the whole batch until no word is the sentinel (one L2 round trip per poll, not per word)
        for (long spins = 0;; ++spins) {
          bool miss = false;
#pragma unroll
          for (int j = 0; j < kB; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              vals[j][q] = c0 + j < p.nc - 1 ? ld_relaxed_u32(slots + (size_t)(c0 + j) * 128 + q * 32 + lane) : 0u;
              miss |= vals[j][q] == kSent;
            }
          if (!__any_sync(0xffffffffu, miss)) break;
          if (spins > (1L << 24)) __trap();                 // a chunk never arrived: fail loudly
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          if (c0 + j >= p.nc - 1) break;
#pragma unroll
          for (int q = 0; q < 4; ++q) tot[q] += __uint_as_float(vals[j][q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        tot[q] += mine[q];
        if (q * 32 + lane < R) yrow[q * 32 + lane] = tot[q];
      }
      for (int cc = 0; cc < p.nc - 1; ++cc)
#pragma unroll
        for (int q = 0; q < 4; ++q) reinterpret_cast<unsigned int*>(slots)[(size_t)cc * 128 + q * 32 + lane] = kSent;
      if (p.ts && lane == 0) {
        unsigned long long* tsw = p.ts + ((size_t)blockIdx.x * kWarps + wib) * 8;
        tsw[5] += gtime() - tr0;
        tsw[6] += 1;
      }
    }
    PTS(3, gtime());
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int gq = lane >> 2, c4 = lane & 3;
  const int u_w = wib >> 2, pr_w = wib & 3;          // unit of the item, tile pair of the unit
  asm volatile("griddepcontrol.wait;" ::: "memory");   // activations from here
  {
    // stage the activation planes and scales in shared memory (named barrier: consumers only)
    const int nx = p.NG * p.l * 4;
    const uint4* src = reinterpret_cast<const uint4*>(p.xplanes);
    uint4* dst = reinterpret_cast<uint4*>(s_xp);
    for (int i = threadIdx.x; i < nx / 4; i += kCons * 32) dst[i] = __ldg(src + i);
    for (int i = threadIdx.x; i < p.NG; i += kCons * 32) s_xs[i] = __ldg(p.xscales + i);
    asm volatile("bar.sync 1, %0;" ::"r"(kCons * 32) : "memory");
  }
  const int j0 = 2 * c4, j1 = 2 * c4 + 1;
  const int al0 = j0 < p.l - 1 ? (1 << j0) : (j0 == p.l - 1 ? -(1 << j0) : 0);
  const int al1 = j1 < p.l - 1 ? (1 << j1) : (j1 == p.l - 1 ? -(1 << j1) : 0);
  const int kappa = al0 != 0 ? al1 / al0 : 0;
  const float lane_scale = (float)al0 * (1.0f / 128.0f);
  const int magic = 0x4B400000;
  const uint32_t xmask = gq < p.l ? 0xffffffffu : 0u;
  const int xoff = gq < p.l ? gq * 4 + c4 : 0;
  const int swz_a = chunk_swizzle(K, gq), swz_b = chunk_swizzle(K, gq + 8);

  for (int it = 0;; ++it) {
    const int slot = it % p.S;
    mbar_wait(full_bar + slot, (it / p.S) & 1);
    if (it == 0) PTS(1, gtime());
    const int v = s_hdr[slot];
    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    if (v >= 0) {
      const int rb = v / p.nc, c = v - rb * p.nc;
      const int g0 = c * kUPS, ng = min(kUPS, p.NG - g0);
      const int R = rb < p.n_full ? 128 : p.tail_rows;
      const int g = g0 + u_w;
      if (u_w < ng && 32 * pr_w < R) {
        const uint8_t* un = stages + (size_t)slot * p.stage_bytes + (size_t)u_w * R * (16 * K + 5);
        // B operand for group g: activation plane gq, word c4, bit-sliced and pre-scaled by 2^(7-s)
        const uint32_t X = s_xp[g * p.l * 4 + xoff] & xmask;
        const float sx = s_xs[g];
        uint32_t Bq[4][2];
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          Bq[pr][0] = bslice(X, 2 * pr);
          Bq[pr][1] = bslice(X, 2 * pr + 1);
        }
        const bool two = 32 * pr_w + 16 < R;            // the pair's second tile exists (tail blocks)
        uint32_t w[2][2 * K];
        uint32_t sb0[2], sb1[2];
        float2 r2[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r0 = 32 * pr_w + 16 * j + (j == 1 && !two ? -16 : 0);   // re-read tile 0 (result dropped)
          const uint8_t* ra = un + (size_t)(r0 + gq) * 16 * K + 4 * c4;
          const uint8_t* rb8 = ra + 8 * 16 * K;
#pragma unroll
          for (int t = 0; t < K; ++t) {
            w[j][2 * t] = *reinterpret_cast<const uint32_t*>(ra + 16 * (t ^ swz_a));
            w[j][2 * t + 1] = *reinterpret_cast<const uint32_t*>(rb8 + 16 * (t ^ swz_b));
          }
          sb0[j] = *reinterpret_cast<const uint32_t*>(un + (size_t)R * 16 * K + (r0 + gq) * 4);
          sb1[j] = *reinterpret_cast<const uint32_t*>(un + (size_t)R * 16 * K + (r0 + gq + 8) * 4);
          r2[j] = make_float2(s_rat[un[(size_t)R * (16 * K + 4) + r0 + gq]], s_rat[un[(size_t)R * (16 * K + 4) + r0 + gq + 8]]);
        }
        int D[2][K][4];
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          const uint32_t m0 = 0x01010101u << (2 * pr), m1 = 0x01010101u << (2 * pr + 1);
#pragma unroll
          for (int t = 0; t < K; ++t)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint32_t a0 = w[j][2 * t] & m0, a1 = w[j][2 * t + 1] & m0;
              const uint32_t a2 = w[j][2 * t] & m1, a3 = w[j][2 * t + 1] & m1;
              if (pr == 0)
                mma_u8(D[j][t], a0, a1, a2, a3, Bq[pr][0], Bq[pr][1], 0, 0, 0, 0);
              else
                mma_u8(D[j][t], a0, a1, a2, a3, Bq[pr][0], Bq[pr][1], D[j][t][0], D[j][t][1], D[j][t][2], D[j][t][3]);
            }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (DEBUG) {
            if (j == 1 && !two) continue;
            const int r0w = 128 * rb + 32 * pr_w + 16 * j + gq;
#pragma unroll
            for (int t = 0; t < K; ++t)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                int32_t* dst = p.P + (((size_t)(r0w + 8 * h) * p.NG + g) * K + t) * p.l;
                if (j0 < p.l) dst[j0] = D[j][t][2 * h] >> 7;
                if (j1 < p.l) dst[j1] = D[j][t][2 * h + 1] >> 7;
              }
          } else {
            const float2 s2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] & 0xffffu))),
                                          __half2float(__ushort_as_half((unsigned short)(sb1[j] & 0xffffu))));
            const float2 b2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] >> 16))),
                                          __half2float(__ushort_as_half((unsigned short)(sb1[j] >> 16))));
            // f_t = 128 (P_2c + kappa P_2c+1) for rows (gq, gq+8), exact; Horner over t in fp32x2
            float2 Ph = __fadd2_rn(make_float2(__int_as_float(imad(imad(D[j][K - 1][1], kappa, D[j][K - 1][0]), p.one, magic)),
                                               __int_as_float(imad(imad(D[j][K - 1][3], kappa, D[j][K - 1][2]), p.one, magic))),
                                   make_float2(-12582912.0f, -12582912.0f));
            float2 U = Ph;
#pragma unroll
            for (int t = K - 2; t >= 0; --t) {
              const float2 f = __fadd2_rn(make_float2(__int_as_float(imad(imad(D[j][t][1], kappa, D[j][t][0]), p.one, magic)),
                                                      __int_as_float(imad(imad(D[j][t][3], kappa, D[j][t][2]), p.one, magic))),
                                          make_float2(-12582912.0f, -12582912.0f));
              Ph = __ffma2_rn(Ph, r2[j], f);
              U = __fadd2_rn(U, f);
            }
            const float2 vv = __ffma2_rn(s2, Ph, __fmul2_rn(b2, U));
            acc[j] = (j == 1 && !two) ? make_float2(0.f, 0.f) : __fmul2_rn(make_float2(sx, sx), vv);
          }
        }
      }
    }
    // release the weight stage
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar + slot);
    if (DEBUG) {
      if (v < 0) break;
      continue;
    }
    // quad-reduce the rows of the tile pair and hand them to the flush warp
    float x[4] = {acc[0].x * lane_scale, acc[0].y * lane_scale, acc[1].x * lane_scale, acc[1].y * lane_scale};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[q] += __shfl_xor_sync(0xffffffffu, x[q], 1);
      x[q] += __shfl_xor_sync(0xffffffffu, x[q], 2);
    }
    const int ps = it % kPS;
    if (it >= kPS) mbar_wait(pempty_bar + ps, ((it / kPS) - 1) & 1);
    if (c4 == 0) {
      float* dst = s_part + ((size_t)ps * kCons + wib) * 32;
      dst[gq] = x[0];                                    // tile 2p row gq
      dst[gq + 8] = x[1];                                // tile 2p row gq+8
      dst[16 + gq] = x[2];                               // tile 2p+1
      dst[16 + gq + 8] = x[3];
    }
    if (wib == 0 && lane == 0) s_phdr[ps] = v;
    __syncwarp();
    if (lane == 0) mbar_arrive(pfull_bar + ps);
    if (v < 0) break;
  }
  PTS(2, gtime());
  if (p.ts && lane == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.ts[((size_t)blockIdx.x * kWarps + wib) * 8 + 4] = smid;
  }
}

static int num_sms_pipe() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct PipePlan {
  int NG, nc, n_rb, n_full, tail_rows, n_items, grid, S, stage_bytes, x_bytes, smem;
};

static PipePlan pipe_plan(const sbvr_weights* w, int l) {
  PipePlan pl;
  pl.NG = w->N / kG;
  pl.nc = (pl.NG + kUPS - 1) / kUPS;
  pl.n_full = w->M / kRowBlock;
  pl.tail_rows = w->M % kRowBlock;
  pl.n_rb = pl.n_full + (pl.tail_rows ? 1 : 0);
  pl.n_items = pl.n_rb * pl.nc;
  pl.grid = std::min(num_sms_pipe(), pl.n_items);
  pl.stage_bytes = (kUPS * 128 * (16 * w->K + 5) + 127) / 128 * 128;
  pl.x_bytes = (pl.NG * l * 16 + 15) / 16 * 16;
  const int fixed = kPS * kCons * 32 * 4 + pl.x_bytes + (pl.NG * 4 + 15) / 16 * 16;
  const int budget = 227 * 1024 - 4096;                // static smem + slack
  pl.S = std::min(kMaxStages, (budget - fixed) / pl.stage_bytes);
  pl.smem = pl.S * pl.stage_bytes + fixed;
  return pl;
}

template <int K, bool DEBUG>
static cudaError_t launch_pipe_k(const PipeParams& p, int grid, int smem, cudaStream_t st) {
  static int attr_set = 0;
  if (attr_set < smem) {
    cudaError_t e = cudaFuncSetAttribute(gemv_pipe_kernel<K, DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPipeThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemv_pipe_kernel<K, DEBUG>, p);
}

template <bool DEBUG>
static cudaError_t launch_pipe_any(int K, const PipeParams& p, int grid, int smem, cudaStream_t st) {
  switch (K) {
    case 1: return launch_pipe_k<1, DEBUG>(p, grid, smem, st);
    case 2: return launch_pipe_k<2, DEBUG>(p, grid, smem, st);
    case 3: return launch_pipe_k<3, DEBUG>(p, grid, smem, st);
    case 4: return launch_pipe_k<4, DEBUG>(p, grid, smem, st);
    case 5: return launch_pipe_k<5, DEBUG>(p, grid, smem, st);
    case 6: return launch_pipe_k<6, DEBUG>(p, grid, smem, st);
    case 7: return launch_pipe_k<7, DEBUG>(p, grid, smem, st);
    default: return launch_pipe_k<8, DEBUG>(p, grid, smem, st);
  }
}

}  // namespace

// [ticket: 16 B][partial slots: n_rb x nc x 128 floats], all 0xFF at rest (sbvr_workspace_init)
size_t pipe_workspace_bytes(const sbvr_weights* w) {
  const int NG = w->N / kG, nc = (NG + kUPS - 1) / kUPS;
  const int n_rb = (w->M + kRowBlock - 1) / kRowBlock;
  return 16 + (size_t)n_rb * nc * 128 * sizeof(float);
}

bool pipe_supported(const sbvr_weights* w, const sbvr_act* x) {
  if (x->kind != SBVR_ACT_SBVR) return false;
  const PipePlan pl = pipe_plan(w, x->l);
  return pl.S >= 2;
}

sbvr_status launch_gemv_pipe(const sbvr_weights* w, const sbvr_act* x, float* y, void* ws, int32_t* P_debug,
                             cudaStream_t st) {
  const PipePlan pl = pipe_plan(w, x->l);
  if (pl.S < 2) return set_error(SBVR_ERR_UNSUPPORTED, "gemv_pipe: activation planes too large for shared memory");
  PipeParams p;
  p.units = w->data;
  p.ratio_pow = w->ratio_pow;
  p.xplanes = static_cast<const uint32_t*>(x->data);
  p.xscales = x->scales;
  p.Y = y;
  p.P = P_debug;
  p.ticket = reinterpret_cast<unsigned int*>(ws);
  p.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 16);
  p.M = w->M; p.N = w->N; p.l = x->l; p.n_ratio = w->n_ratio;
  p.n_full = pl.n_full; p.tail_rows = pl.tail_rows; p.n_rb = pl.n_rb; p.NG = pl.NG; p.nc = pl.nc;
  p.n_items = pl.n_items; p.S = pl.S; p.stage_bytes = pl.stage_bytes; p.x_bytes = pl.x_bytes;
  p.one = 1;
  const char* tsp = getenv("SBVR_TS_PTR");
  p.ts = tsp ? reinterpret_cast<unsigned long long*>(strtoull(tsp, nullptr, 0)) : nullptr;
  cudaError_t e = P_debug ? launch_pipe_any<true>(w->K, p, pl.grid, pl.smem, st)
                          : launch_pipe_any<false>(w->K, p, pl.grid, pl.smem, st);
  if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "gemv_pipe setup: %s", cudaGetErrorString(e));
  return check_launch("gemv_pipe_kernel");
}

}  // namespace sbvr
