// gemv_group.cu -- grouped SBVR GEMV: several independent batch-1 GEMVs y_p = W_p x_p (§4.4, P:245-251;
// SBVR-x, the AND+popcount form of gemv_mma.cuh) in ONE persistent launch (sbvr_gemv_group, include/sbvr.h).
//
// Why: a batch-1 GEMV of a decoder layer moves 2-32 MB, so a launch that streams it at the core rate lasts only
// 3-20 us, and every launch pays a fixed cost that does not shrink with the matrix -- first bytes ~2 us after the
// CTA starts, split-K combine, CTA tail spread, the next launch's griddepcontrol.wait (profiles/r02_phase_step.txt:
// ~45% of the 4-launch step).  Here the problems' units are concatenated into one global unit sequence
//     problem 0's units (band-major, as in HBM) | problem 1's units | ...
// which is split into balanced contiguous CTA ranges and warp ranges exactly like gemv_mma's single problem; a
// warp's private TMA ring simply runs on across problem boundaries (the next matrix's first records are in flight
// while the current one is finishing), and the fixed costs are paid once per group, not once per matrix.
//
// Arithmetic per (row, group) is the MMA kernel's, bit for bit: A = plane word & (0x01010101 << s), B = activation
// plane j bit-sliced x 2^(7-s), mma.m16n8k32.u8 accumulates 128 P_tj, epilogue u = D0 + kappa D1, exact int->float,
// Horner over t in fp32x2, y += s_x (s sum_t r^t u_t + b sum_t u_t).  A band (64 rows of one matrix) shared by
// several warps / CTAs is combined by the same deterministic last-arriver reduction (smem counter in warp order;
// global counter + sentinel-validated slots in CTA order), so every y is bit-identical to sbvr_gemv on the MMA
// kernel when the band split is the same -- and deterministic in any case.  Restrictions (checked by the ABI):
// T = 1, SBVR-x, SBVR_META_GROUP, K in 2..4 and the same for every problem, M % 128 == 0, 1..8 problems.
#include "gemv_mma.cuh"

namespace sbvr {
namespace grp {
using namespace mma;

constexpr int kMaxProb = SBVR_GROUP_MAX;
constexpr int NB = 4;                     // tiles (16 rows) per band

struct GProb {
  const uint8_t* units;     // unit records of W_p (sbvr.h; full 128-row blocks only)
  const uint32_t* xplanes;  // [NG][l][4]
  const float* xscales;     // [NG]
  float* Y;                 // [M]
  int NG;                   // groups per row
  int bbase;                // first global band of this problem
  int ubase;                // first global unit of this problem
};

struct GroupParams {
  GProb pr[kMaxProb];
  const float* ratio_pow[kMaxProb];   // [n_ratio][K] per problem
  int n_ratio[kMaxProb];
  int np;                   // problems
  int Us;                   // total units
  int C, qq, rr;            // CTAs and the unit partition over CTAs
  int l, one;
  float* ws_part;           // [CTA][2][64] fp32 partials of a CTA's first / last band (kSentinel at rest)
  unsigned int* ws_cnt;     // [global band] arrival counters (0xFFFFFFFF at rest)
};

// position in the global unit sequence: problem p, global band b, group g
struct Pos {
  int p, b, g;
};
__device__ __forceinline__ Pos pos_of(const GroupParams& P, int u) {
  int p = 0;
#pragma unroll 1
  while (p + 1 < P.np && u >= P.pr[p + 1].ubase) ++p;
  const int loc = u - P.pr[p].ubase, NG = P.pr[p].NG;
  return Pos{p, P.pr[p].bbase + loc / NG, loc % NG};
}
__device__ __forceinline__ void advance(const GroupParams& P, Pos& q) {
  if (++q.g == P.pr[q.p].NG) {
    q.g = 0;
    ++q.b;
    if (q.p + 1 < P.np && q.b == P.pr[q.p + 1].bbase) ++q.p;
  }
}
// first global unit of global band b (of problem p)
__device__ __forceinline__ int band_first_unit(const GroupParams& P, int p, int b) {
  return P.pr[p].ubase + (b - P.pr[p].bbase) * P.pr[p].NG;
}

template <int K>
__device__ __forceinline__ void issue_gunit(uint8_t* slot, uint64_t* bar, const GroupParams& P, const Pos& q, int i0,
                                            int i1) {
  using Gm = Geom<K, NB, false>;
  const int NG = P.pr[q.p].NG;
  const int lb = q.b - P.pr[q.p].bbase;
  const int rb = lb >> 1, h = lb & 1;
  constexpr int R = 128;
  const size_t ub = (size_t)R * (16 * K + 5);
  const uint8_t* u = P.pr[q.p].units + ((size_t)rb * NG + q.g) * ub;
  const int r0 = 64 * h + 16 * i0, nt = i1 - i0;
  mbar_expect_tx(bar, nt * (Gm::kTileBytes + 64 + 16));
  bulk_g2s(slot + i0 * Gm::kTileBytes, u + (size_t)r0 * 16 * K, nt * Gm::kTileBytes, bar);
  bulk_g2s(slot + Gm::kPlaneBytes + 64 * i0, u + (size_t)R * 16 * K + 4 * r0, nt * 64, bar);
  bulk_g2s(slot + Gm::kPlaneBytes + Gm::kSbBytes + 16 * i0, u + (size_t)R * (16 * K + 4) + r0, nt * 16, bar);
}

template <int K>
__global__ void __launch_bounds__(kImmaWarps * 32, SBVR_MMA_CTAS_PER_SM) gemv_group_kernel(GroupParams P) {
  using Gm = Geom<K, NB, false>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float s_rat[kMaxProb * 64];          // r_i of every problem (Horner of sum_t r^t u_t)
  __shared__ uint64_t s_bar[kImmaWarps][kSlots];
  __shared__ unsigned int s_cnt[2 * kImmaWarps];  // warps done with a band, by (first warp, its first/last band)
  __shared__ int s_fb[kImmaWarps];                // first global band of each warp
  __shared__ int s_lb[kImmaWarps];                // last global band of each warp (-1: no tiles)
  float* s_part = reinterpret_cast<float*>(smem + kImmaWarps * Gm::kWarpBytes);   // [warps][2][64]
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int cta = blockIdx.x;
  const int V0 = cta * P.qq + min(cta, P.rr);
  const int V1 = V0 + P.qq + (cta < P.rr ? 1 : 0);
  // this CTA's tiles split over its warps at single-tile granularity: warp w takes tiles [T0, T1)
  const int nTc = (V1 - V0) * NB;
  const int tq = nTc / kImmaWarps, tr = nTc % kImmaWarps;
  const int T0 = wib * tq + min(wib, tr), T1 = T0 + tq + (wib < tr ? 1 : 0);
  const int n_mine = T1 > T0 ? (T1 - 1) / NB - T0 / NB + 1 : 0;
  const int uf = V0 + T0 / NB;
  auto tiles_of = [&](int k, int& i0, int& i1) {
    i0 = k == 0 ? T0 % NB : 0;
    i1 = k == n_mine - 1 ? (T1 - 1) % NB + 1 : NB;
  };
  uint8_t* ring = smem + wib * Gm::kWarpBytes;
  uint64_t* bars = s_bar[wib];
  Pos iq{0, 0, 0};                                  // lane 0: the next unit to fetch
  if (n_mine > 0) iq = pos_of(P, uf);
  auto issue_next = [&](uint8_t* slot_ptr, uint64_t* bar, int kk) {
    int i0, i1;
    tiles_of(kk, i0, i1);
    issue_gunit<K>(slot_ptr, bar, P, iq, i0, i1);
    advance(P, iq);
  };
  if (n_mine > 0 && lane == 0) {
    // weights are immutable: their copies start before we wait for the previous kernel
#pragma unroll
    for (int s2 = 0; s2 < kSlots; ++s2) mbar_init(bars + s2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s2 = 0; s2 < kSlots; ++s2)
      if (s2 < n_mine) issue_next(ring + s2 * Gm::kSlotBytes, bars + s2, s2);
  }
  for (int i = threadIdx.x; i < kMaxProb * 64; i += blockDim.x) {
    const int pp = i >> 6, ri = i & 63;
    s_rat[i] = (pp < P.np && ri < P.n_ratio[pp] && K >= 2) ? P.ratio_pow[pp][ri * K + 1] : 0.f;
  }
  for (int i = threadIdx.x; i < 2 * kImmaWarps; i += blockDim.x) s_cnt[i] = 0u;
  if (threadIdx.x < kImmaWarps) {
    const int w2 = threadIdx.x;
    const int t0 = w2 * tq + min(w2, tr), t1 = t0 + tq + (w2 < tr ? 1 : 0);
    s_fb[w2] = t1 > t0 ? pos_of(P, V0 + t0 / NB).b : 0x7fffffff;
    s_lb[w2] = t1 > t0 ? pos_of(P, V0 + (t1 - 1) / NB).b : -1;
  }
  __syncthreads();
  if (n_mine <= 0) return;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // activations / workspace / y from here

  // lane constants (Eq. 12: alpha_j = 2^j, alpha_{l-1} = -2^(l-1); MMA columns j0 = 2c, j1 = 2c+1)
  const int j0 = 2 * c, j1 = 2 * c + 1;
  const int al0 = j0 < P.l - 1 ? (1 << j0) : (j0 == P.l - 1 ? -(1 << j0) : 0);
  const int al1 = j1 < P.l - 1 ? (1 << j1) : (j1 == P.l - 1 ? -(1 << j1) : 0);
  const int kappa = al0 != 0 ? al1 / al0 : 0;
  const float lane_scale = (float)al0 * (1.0f / 128.0f);
  const int magic = 0x4B400000;
  const float2 cmagic = make_float2(12582912.0f, 12582912.0f);
  const uint32_t xmask = gq < P.l ? 0xffffffffu : 0u;
  const int xoff = gq < P.l ? gq * 4 + c : 0;
  const int xstride = P.l * 4;
  const int swz_a = chunk_swizzle(K, gq), swz_b = chunk_swizzle(K, gq + 8);

  float2 acc[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) acc[i] = make_float2(0.f, 0.f);

  Pos q = pos_of(P, uf);
  int slot = 0;
  uint32_t phase = 0;
  uint32_t Xn = __ldg(P.pr[q.p].xplanes + (size_t)q.g * xstride + xoff);
  float sxn = __ldg(P.pr[q.p].xscales + q.g);

  for (int k = 0; k < n_mine; ++k) {
    // ---- B operand for group g: activation plane gq, word c, bit-sliced and pre-scaled by 2^(7-s)
    uint32_t Bq[4][2];
    const float sx = sxn;
    {
      const uint32_t X = Xn & xmask;
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        Bq[pr][0] = bslice(X, 2 * pr);
        Bq[pr][1] = bslice(X, 2 * pr + 1);
      }
    }
    const int rat_off = q.p * 64;
    Pos qn = q;
    advance(P, qn);
    int ti0, ti1;
    tiles_of(k, ti0, ti1);
    const bool has_next = k + 1 < n_mine;
    {
      const Pos& qp = has_next ? qn : q;
      Xn = __ldg(P.pr[qp.p].xplanes + (size_t)qp.g * xstride + xoff);
      sxn = __ldg(P.pr[qp.p].xscales + qp.g);
    }

    uint8_t* sl = ring + slot * Gm::kSlotBytes;
    mbar_wait(bars + slot, phase);

    auto step = [&](auto ptc, const int ib) {
      constexpr int PT = decltype(ptc)::value;
      uint32_t w[PT][2 * K];
      uint32_t sb0[PT], sb1[PT];
      float2 r2[PT];
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        const int i = ib + j;
        const uint8_t* ra = sl + (16 * i + gq) * 16 * K + 4 * c;
        const uint8_t* rb8 = ra + 8 * 16 * K;
#pragma unroll
        for (int t = 0; t < K; ++t) {
          w[j][2 * t] = *reinterpret_cast<const uint32_t*>(ra + 16 * (t ^ swz_a));
          w[j][2 * t + 1] = *reinterpret_cast<const uint32_t*>(rb8 + 16 * (t ^ swz_b));
        }
        sb0[j] = *reinterpret_cast<const uint32_t*>(sl + Gm::kPlaneBytes + (16 * i + gq) * 4);
        sb1[j] = *reinterpret_cast<const uint32_t*>(sl + Gm::kPlaneBytes + (16 * i + gq + 8) * 4);
        r2[j] = make_float2(s_rat[rat_off + sl[Gm::kPlaneBytes + Gm::kSbBytes + 16 * i + gq]],
                            s_rat[rat_off + sl[Gm::kPlaneBytes + Gm::kSbBytes + 16 * i + gq + 8]]);
      }
      // ---- AND + popcount on the tensor pipe: PT x K independent chains (tile, plane) of 4 MMAs
      int D[PT][K][4];
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        const uint32_t m0 = 0x01010101u << (2 * pr), m1 = 0x01010101u << (2 * pr + 1);
#pragma unroll
        for (int t = 0; t < K; ++t)
#pragma unroll
          for (int j = 0; j < PT; ++j) {
            const uint32_t a0 = w[j][2 * t] & m0, a1 = w[j][2 * t + 1] & m0;
            const uint32_t a2 = w[j][2 * t] & m1, a3 = w[j][2 * t + 1] & m1;
            if (pr == 0)
              mma_u8(D[j][t], a0, a1, a2, a3, Bq[pr][0], Bq[pr][1], 0, 0, 0, 0);
            else
              mma_u8(D[j][t], a0, a1, a2, a3, Bq[pr][0], Bq[pr][1], D[j][t][0], D[j][t][1], D[j][t][2], D[j][t][3]);
          }
      }
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        const int i = ib + j;
        const float2 s2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] & 0xffffu))),
                                      __half2float(__ushort_as_half((unsigned short)(sb1[j] & 0xffffu))));
        const float2 b2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] >> 16))),
                                      __half2float(__ushort_as_half((unsigned short)(sb1[j] >> 16))));
        // f_t = 128 (P_2c + kappa P_2c+1) for rows (gq, gq+8), exact; Horner over t in fp32x2
        float2 Ph = __fadd2_rn(make_float2(__int_as_float(imad(imad(D[j][K - 1][1], kappa, D[j][K - 1][0]), P.one, magic)),
                                           __int_as_float(imad(imad(D[j][K - 1][3], kappa, D[j][K - 1][2]), P.one, magic))),
                               make_float2(-cmagic.x, -cmagic.y));
        float2 U = Ph;
#pragma unroll
        for (int t = K - 2; t >= 0; --t) {
          const float2 f = __fadd2_rn(make_float2(__int_as_float(imad(imad(D[j][t][1], kappa, D[j][t][0]), P.one, magic)),
                                                  __int_as_float(imad(imad(D[j][t][3], kappa, D[j][t][2]), P.one, magic))),
                                      make_float2(-cmagic.x, -cmagic.y));
          Ph = __ffma2_rn(Ph, r2[j], f);
          U = __fadd2_rn(U, f);
        }
        const float2 v = __ffma2_rn(s2, Ph, __fmul2_rn(b2, U));
        acc[i] = __ffma2_rn(make_float2(sx, sx), v, acc[i]);
      }
    };
#pragma unroll
    for (int ib = 0; ib < NB; ib += 2) {
      const bool in0 = ib >= ti0 && ib < ti1;
      const bool in1 = ib + 1 >= ti0 && ib + 1 < ti1;
      if (in0 && in1) step(std::integral_constant<int, 2>{}, ib);
      else if (in0) step(std::integral_constant<int, 1>{}, ib);
      else if (in1) step(std::integral_constant<int, 1>{}, ib + 1);
    }

    // ---- release the slot and refill it with this warp's unit k + kSlots (possibly the next matrix's)
    __syncwarp();
    if (lane == 0 && k + kSlots < n_mine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_next(sl, bars + slot, k + kSlots);
    }
    if (++slot == kSlots) { slot = 0; phase ^= 1u; }

    // ---- leaving band q.b: warp-level then CTA-level combine (see gemv_mma.cuh; bands are global here)
    const int b = q.b;
    if (!has_next || qn.b != b) {
      const unsigned int holders =
          __ballot_sync(0xffffffffu, lane < kImmaWarps && s_fb[min(lane, kImmaWarps - 1)] <= b &&
                                         s_lb[min(lane, kImmaWarps - 1)] >= b);
      const int wf = __ffs(holders) - 1, wl = 31 - __clz(holders);
      const int ub0 = band_first_unit(P, q.p, b), ub1 = ub0 + P.pr[q.p].NG;   // the band's global units
      const bool shared = V0 > ub0 || V1 < ub1;                                // other CTAs hold units of b
      float* sp = s_part + ((size_t)wib * 2 + (b == s_fb[wib] ? 0 : 1)) * 64;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        float x0 = acc[i].x * lane_scale, x1 = acc[i].y * lane_scale;
        x0 += __shfl_xor_sync(0xffffffffu, x0, 1);
        x1 += __shfl_xor_sync(0xffffffffu, x1, 1);
        x0 += __shfl_xor_sync(0xffffffffu, x0, 2);
        x1 += __shfl_xor_sync(0xffffffffu, x1, 2);
        if (c == 0) {
          sp[16 * i + gq] = x0;
          sp[16 * i + gq + 8] = x1;
        }
        acc[i] = make_float2(0.f, 0.f);
      }
      bool last = true;
      if (wf != wl) {
        __syncwarp();
        unsigned int old = 0;
        const int fbf = s_fb[wf];
        if (lane == 0) {
          __threadfence_block();
          old = atomicAdd(&s_cnt[wf * 2 + (b == fbf ? 0 : 1)], 1u);
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        last = old == (unsigned int)(wl - wf);
      }
      if (last) {
        __syncwarp();
        __threadfence_block();
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float sum = 0.f;
          for (int w2 = wf; w2 <= wl; ++w2)               // contributing warps, in warp order
            sum += s_part[((size_t)w2 * 2 + (b == s_fb[w2] ? 0 : 1)) * 64 + lane + 32 * h];
          v[h] = sum;
        }
        float* Yp = P.pr[q.p].Y + 64 * (b - P.pr[q.p].bbase);
        if (!shared) {
#pragma unroll
          for (int h = 0; h < 2; ++h) Yp[lane + 32 * h] = v[h];
        } else {
          // last-arriver reduction over the CTAs holding units of b (deterministic CTA order, no waiting on
          // another CTA's progress: see gemv_mma.cuh)
          const int myslot = V0 >= ub0 ? 0 : 1;
          float* part = P.ws_part + ((size_t)cta * 2 + myslot) * 64;
#pragma unroll
          for (int h = 0; h < 2; ++h) __stcg(part + lane + 32 * h, v[h]);
          __syncwarp();
          const int c0 = unit_owner(ub0, P.qq, P.rr);
          const int c1 = unit_owner(ub1 - 1, P.qq, P.rr);
          unsigned int old = 0;
          if (lane == 0) old = atomicAdd(P.ws_cnt + b, 1u);
          old = __shfl_sync(0xffffffffu, old, 0);
          if (old + 2u == (unsigned int)(c1 - c0 + 1)) {
            float sum[2] = {0.f, 0.f};
            for (int cb = c0; cb <= c1; cb += kSumBatchMax) {
              uint32_t vals[kSumBatchMax][2];
              for (long spins = 0;; ++spins) {       // reload the batch until no word is the sentinel
                bool miss = false;
#pragma unroll
                for (int j = 0; j < kSumBatchMax; ++j) {
                  const int cc = cb + j;
                  const int v0c = cc * P.qq + min(cc, P.rr);             // first unit of CTA cc
                  const float* src = P.ws_part + ((size_t)cc * 2 + (v0c >= ub0 ? 0 : 1)) * 64;
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    vals[j][h] = cc > c1 ? 0u : cc == cta ? __float_as_uint(v[h]) : ld_relaxed(src + lane + 32 * h);
                    miss |= vals[j][h] == kSentinel;
                  }
                }
                if (!__any_sync(0xffffffffu, miss)) break;
                if (spins > (1L << 26)) __trap();    // stores already issued never landed: fail loudly
              }
#pragma unroll
              for (int j = 0; j < kSumBatchMax; ++j) {
                if (cb + j > c1) break;
#pragma unroll
                for (int h = 0; h < 2; ++h) sum[h] += __uint_as_float(vals[j][h]);
              }
            }
            for (int cc = c0; cc <= c1; ++cc) {
              const int v0c = cc * P.qq + min(cc, P.rr);
              unsigned int* dst = reinterpret_cast<unsigned int*>(P.ws_part) + ((size_t)cc * 2 + (v0c >= ub0 ? 0 : 1)) * 64;
#pragma unroll
              for (int h = 0; h < 2; ++h) dst[lane + 32 * h] = kSentinel;
            }
            if (lane == 0) P.ws_cnt[b] = kSentinel;
#pragma unroll
            for (int h = 0; h < 2; ++h) Yp[lane + 32 * h] = sum[h];
          }
        }
      }
    }
    q = qn;
  }
}

// ------------------------------------------------------------------ host side
static int group_num_sms() {
  static int n[64] = {0};
  const int dev = cur_device();
  if (dev < 0 || dev >= 64) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

struct GroupPlan {
  int n_bands, Us, C;
};
static GroupPlan group_plan(const sbvr_gemv_problem* pr, int n) {
  GroupPlan g{0, 0, 0};
  for (int i = 0; i < n; ++i) {
    g.n_bands += pr[i].w.M / 64;
    g.Us += (pr[i].w.M / 64) * (pr[i].w.N / kG);
  }
  int C = group_num_sms() * SBVR_MMA_CTAS_PER_SM;
  const int cap = (g.Us + kMinUnitsPerCta - 1) / kMinUnitsPerCta;
  g.C = C > cap ? cap : (C < 1 ? 1 : C);
  return g;
}
static size_t group_cnt_bytes(const GroupPlan& g) { return ((size_t)(g.n_bands + 1) * 4 + 255) / 256 * 256; }

template <int K>
static cudaError_t launch_group_k(const GroupParams& P, cudaStream_t st) {
  const int smem = kImmaWarps * Geom<K, NB, false>::kWarpBytes + kImmaWarps * 2 * 64 * 4;
  static int attr_set[64] = {0};
  const int dev = cur_device();
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemv_group_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.C);
  cfg.blockDim = dim3(kImmaWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemv_group_kernel<K>, P);
}

}  // namespace grp

size_t group_workspace_bytes(const sbvr_gemv_problem* pr, int n) {
  const grp::GroupPlan g = grp::group_plan(pr, n);
  return grp::group_cnt_bytes(g) + (size_t)g.C * 2 * 64 * sizeof(float);
}

sbvr_status launch_gemv_group(const sbvr_gemv_problem* pr, int n, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace grp;
  const GroupPlan g = group_plan(pr, n);
  const size_t need = group_workspace_bytes(pr, n);
  if (ws_bytes < need)
    return set_error(SBVR_ERR_WORKSPACE, "gemv_group: workspace %zu bytes < required %zu", ws_bytes, need);
  GroupParams P = {};
  int bb = 0, uu = 0;
  for (int i = 0; i < n; ++i) {
    P.pr[i].units = pr[i].w.data;
    P.pr[i].xplanes = static_cast<const uint32_t*>(pr[i].x.data);
    P.pr[i].xscales = pr[i].x.scales;
    P.pr[i].Y = pr[i].y;
    P.pr[i].NG = pr[i].w.N / kG;
    P.pr[i].bbase = bb;
    P.pr[i].ubase = uu;
    P.ratio_pow[i] = pr[i].w.ratio_pow;
    P.n_ratio[i] = pr[i].w.n_ratio;
    bb += pr[i].w.M / 64;
    uu += (pr[i].w.M / 64) * (pr[i].w.N / kG);
  }
  P.np = n;
  P.Us = g.Us;
  P.C = g.C;
  P.qq = g.Us / g.C;
  P.rr = g.Us % g.C;
  P.l = pr[0].x.l;
  P.one = 1;
  P.ws_cnt = reinterpret_cast<unsigned int*>(ws);
  P.ws_part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + group_cnt_bytes(g));
  cudaError_t e;
  switch (pr[0].w.K) {
    case 2: e = launch_group_k<2>(P, st); break;
    case 3: e = launch_group_k<3>(P, st); break;
    default: e = launch_group_k<4>(P, st); break;
  }
  if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "gemv_group setup: %s", cudaGetErrorString(e));
  return check_launch("gemv_group_kernel");
}

}  // namespace sbvr
