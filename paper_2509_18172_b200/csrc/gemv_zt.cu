// gemv_zt.cu -- SBVR GEMV for a batch of T tokens on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, accumulators in tensor memory): PAPER.md §4.4 for every token of the batch,
// with one pass over the weights for up to 32 tokens (north star "batched (>1 token) variant ...
// dense contraction", "leverage tensor cores ... amortizing the
// dequantization overhead across multiple tokens").
//
// The z-column form.  For weight plane t of a group and token tau the paper's partial
//     T_t = sum_j alpha_j popc(beta_t AND d_j)     (alpha_j = 2^j, alpha_{l-1} = -2^(l-1), Eq. 12)
// equals sum_e beta_t[e] * z_e with z_e = sum_j alpha_j d_j[e] the token's int8 activation code, so
// one u8 x s8 MMA with A = the plane bits as bytes 0/1 (M = 128 rows, K = 32 elements) and B = z
// (N = tokens) accumulates T_t exactly for 128 rows x N tokens.  Then, per (row, group, token),
//     y += s_x * sum_t c_t T_t,   c_t = s r^t + b                 (Eq. 4, fp32)
//
// Why this shape on sm_100a (profiles/r02_tc_rate_issuers.jsonl): a small-N tcgen05.mma holds its
// issuing warp for ~54 cycles, so one issuer caps an SM near 128x32 A bytes per 54 cycles; four issuer
// warps (one per weight plane) bring an M=128 N<=32 MMA to ~14-16 SM-cycles, at the N/2 floor.  A is
// kept in tensor memory (from shared memory the SM's shared-memory bandwidth paces it at ~38 cycles).
//
// CTA = one SM (persistent over a balanced contiguous range of (128-row block, group) units, the
// unit records of include/sbvr.h), 13 warps:
//   warp 12        producer: cp.async.bulk of whole unit records into a 4-slot ring (weights only,
//                  so it runs ahead of griddepcontrol.wait -- programmatic dependent launch)
//   warps 8..11    MMA issuers, one per weight plane t: 4 MMAs (K = 32 x 4 = 128 elements) into D_t
//   warps 0..7     workers, thread = row = TMEM lane, two warps per lane quarter:
//                  - B: the unit's group of z for N tokens, rebuilt from the SBVR-x planes (delta-swap
//                    8x8 bit transposes) into a 2-slot shared-memory ring (canonical K-major layout)
//                  - A: each row's plane words expanded to bytes (w >> s) & 0x01010101 -> tcgen05.st
//                    into a 2-slot tensor-memory ring per plane
//                  - epilogue of the previous unit: tcgen05.ld of D_t, fp32 sum_t c_t T_t, y += s_x ...
// Row blocks shared with other CTAs are combined by the last-arriving CTA in CTA order (deterministic,
// no CTA waits for another: the same sentinel-validated scheme as gemv_mma).
#include <cstdlib>

#include "ptx_sm100.cuh"
#include "sbvr_internal.cuh"

namespace sbvr {
namespace zt {

using namespace ptx;

constexpr int kSlots = 4;          // TMA ring depth (unit records)
constexpr int kExpandWarps = 16;   // A expansion (one plane each) + B build + coefficients: 4 per TMEM lane quarter
constexpr int kEpiWarps = 8;       // epilogue (TMEM -> y) and split-K flush: 2 per lane quarter
constexpr int kIssuerWarps = 4;    // MMA issue, one per weight plane (K <= 4)
constexpr int kThreads = (kExpandWarps + kEpiWarps + kIssuerWarps) * 32;
constexpr int kRing = 8;           // depth of the per-unit coefficient / token-scale ring (expansion -> epilogue)
constexpr int kMaxPlanes = 4;
constexpr int kMaxNT = 32;         // tokens per weight pass
#ifndef ZT_AB_SLOTS
#define ZT_AB_SLOTS 2
#endif
constexpr int kAS = ZT_AB_SLOTS;
#ifndef ZT_MIN_UNITS
#define ZT_MIN_UNITS 8
#endif   // A (tensor memory) / B (shared memory) slots: units in flight between expansion and MMA
constexpr unsigned int kSentinel = 0xFFFFFFFFu;

struct ZtParams {
  const uint8_t* units;      // unit records (sbvr.h)
  const float* ratio_pow;    // [n_ratio][K]
  const uint32_t* xplanes;   // [ntok][NG][l][4] (this pass)
  const float* xscales;      // [ntok][NG]
  float* Y;                  // [ntok][M] (this pass)
  int32_t* Tdbg;             // debug: T_t integers [M][NG][K][ntok]
  float* ws_part;            // [CTA][2 (first / last row block)][NT][128]
  unsigned int* ws_cnt;      // [row block] arrival counters (0xFFFFFFFF at rest)
  int M, N, l, n_ratio, ntok;
  int n_full, tail_rows;     // full 128-row blocks, rows of the tail block
  int Us, qq, rr;            // units, and their partition over CTAs
  unsigned long long* ts;    // diagnostics (-DSBVR_DIAG, env SBVR_TS_PTR): [CTA][32] per-phase SM-cycle totals
};
#ifndef ZT_CRIT_SPIN
#define ZT_CRIT_SPIN 1    // 1: critical-path waits (issuer on A/B ready, expansion on A/B free) spin instead of backing off
#endif
#if ZT_CRIT_SPIN
#define ZT_WAIT_CRIT(bar, ph) mbar_wait(bar, ph)
#else
#define ZT_WAIT_CRIT(bar, ph) mbar_wait_backoff(bar, ph)
#endif
#ifndef ZT_ABL
#define ZT_ABL 0   // ablation bits (diagnostic builds only): 1 no B build, 2 no A expansion, 4 no MMAs, 8 no x loads
#endif
#ifdef SBVR_DIAG
// per-phase SM-cycle totals of one worker thread (warp 0, lane 0) and one issuer (warp 8) per CTA:
// ts[CTA][0..15] worker phases, ts[CTA][16..31] issuer phases (tools/phase_zt.py)
#define PH_DECL unsigned long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long ph_last_ = clock64();
#define PH(s) do { const long long n_ = clock64(); ph_[s] += n_ - ph_last_; ph_last_ = n_; } while (0)
#define PH_DUMP(base) do { if (p.ts && lane == 0) for (int i_ = 0; i_ < 8; ++i_) \
                             p.ts[(size_t)blockIdx.x * 32 + (base) + i_] = ph_[i_]; } while (0)
#else
#define PH_DECL
#define PH(s) do { } while (0)
#define PH_DUMP(base) do { } while (0)
#endif

__device__ __forceinline__ int range_begin(int c, int qq, int rr) { return c * qq + min(c, rr); }
__device__ __forceinline__ int unit_cta(int v, int qq, int rr) {
  const int big = rr * (qq + 1);
  return v < big ? v / (qq + 1) : rr + (v - big) / qq;
}

// w >> s on the FMA pipe (IMAD.HI by 2^(32-s)): the mask that follows runs on the ALU pipe, so the byte
// expansion of A costs one issue slot on each pipe per output word instead of two on the ALU
__device__ __forceinline__ uint32_t shr_fma(uint32_t w, int s) {
  if (s == 0) return w;
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(1u << (32 - s)));
  return r;
}

template <int K, int NT, bool DEBUG>
__global__ void __launch_bounds__(kThreads, 1) gemv_zt_kernel(ZtParams p) {
  static_assert(K >= 1 && K <= kMaxPlanes && NT >= 8 && NT <= kMaxNT, "ZT shape");
  constexpr int kUnitFull = 128 * (16 * K + 5);
  constexpr int kSlotBytes = (kUnitFull + 127) / 128 * 128;
  constexpr int kBBytes = 4 * NT * 32;           // B_q (q = 0..3): NT rows x 32 bytes each
  constexpr int TQ = NT / 2;                     // tokens per epilogue warp (2 per lane quarter)
  constexpr int kDCol = 32 * kAS * K;           // A_t[slot] at 32 (kAS t + slot); D_t[buf] at kDCol + NT (t + K buf)
  // D double-buffered when it fits (MMA(k) need not wait for the epilogue of unit k-1)
  constexpr int kDBuf = kDCol + 2 * K * NT <= 512 ? 2 : 1;
  static_assert(kDCol + K * NT <= 512, "tensor memory: A slots + one D buffer exceed 512 columns");
  constexpr int TC = TQ < 8 ? TQ : 8;            // epilogue token chunk (K x TC registers per TMEM load round)
  constexpr uint32_t kIdesc = (2u << 4) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) | (8u << 24);  // s32 += u8*s8, M=128
  constexpr int kE = kExpandWarps, kP = kEpiWarps;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint8_t* sB = smem + kSlots * kSlotBytes;
  float* s_c = reinterpret_cast<float*>(sB + kAS * kBBytes);      // [kRing][K][128] c_t = s r^t + b per row
  __shared__ float s_rpow[64 * kMaxPlanes];
  __shared__ __align__(8) uint64_t bar_full[kSlots];
  __shared__ __align__(8) uint64_t bar_a[kAS];
  __shared__ __align__(8) uint64_t bar_abfree[kAS];   // MMAs of a unit done (all planes): its A/B slots are free
  __shared__ __align__(8) uint64_t bar_dfull[kMaxPlanes][2];
  __shared__ __align__(8) uint64_t bar_dempty[kMaxPlanes][2];
  __shared__ unsigned int s_rel[kSlots];          // expansion warps done with a ring slot (the last refills it)
  __shared__ uint32_t s_tmem;
  __shared__ unsigned int s_old;
  __shared__ float s_sx[kRing][kMaxNT];           // token scales of a unit's group

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NG = p.N / kG;
  const int cta = blockIdx.x;
  const int V0 = range_begin(cta, p.qq, p.rr);
  const int V1 = range_begin(cta + 1, p.qq, p.rr);
  const int n = V1 - V0;
  const long full_units = (long)p.n_full * NG;
  const uint32_t tail_ub = (uint32_t)p.tail_rows * (16 * K + 5);
  auto unit_src = [&](int u) -> const uint8_t* {
    return u < full_units ? p.units + (size_t)u * kUnitFull
                          : p.units + (size_t)full_units * kUnitFull + (size_t)(u - full_units) * tail_ub;
  };
  auto unit_bytes = [&](int u) -> uint32_t { return u < full_units ? (uint32_t)kUnitFull : tail_ub; };
  auto rows_of = [&](int rb) { return rb < p.n_full ? 128 : p.tail_rows; };

  if (tid == (kE + kP) * 32) {                   // first issuer thread: barriers + the first copies
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&bar_full[s], 1);
      s_rel[s] = 0;
    }
    for (int s = 0; s < kAS; ++s) {
      mbar_init(&bar_a[s], kE);
      mbar_init(&bar_abfree[s], K);
    }
    for (int t = 0; t < kMaxPlanes; ++t)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bar_dfull[t][b], 1);
        mbar_init(&bar_dempty[t][b], kP);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // weights are immutable: their copies start before the previous kernel has finished
    for (int s = 0; s < kSlots && s < n; ++s) {
      mbar_expect_tx(&bar_full[s], unit_bytes(V0 + s));
      bulk_g2s(ring + s * kSlotBytes, unit_src(V0 + s), unit_bytes(V0 + s), &bar_full[s]);
    }
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  for (int i = tid; i < p.n_ratio * K; i += blockDim.x) s_rpow[i] = p.ratio_pow[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp >= kE + kP) {
    // ------------------------------------------------------------ MMA issuer of plane t
    const int t = warp - (kE + kP);
    if (t < K && lane == 0) {
      PH_DECL
      const uint32_t bbase = smem_u32(sB);
      for (int k = 0; k < n; ++k) {
        ZT_WAIT_CRIT(&bar_a[k % kAS], (k / kAS) & 1);           // A_t / B of unit k are in place
        PH(0);
        const int db = k % kDBuf;
        if (k >= kDBuf)                                          // the epilogue has read D_t[db] of unit k - kDBuf
          mbar_wait_backoff(&bar_dempty[t][db], ((k / kDBuf) - 1) & 1);
        tc_fence_after();
        PH(1);
        const uint32_t tA = tmem + 32 * (kAS * t + k % kAS);
        const uint32_t tD = tmem + kDCol + NT * (t + K * db);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (!(ZT_ABL & 4)) mma_i8_ts(tD, tA + 8 * q, smem_desc(bbase + (k % kAS) * kBBytes + q * NT * 32, 128, 256), kIdesc, q);
        mma_commit(&bar_dfull[t][db]);
        mma_commit(&bar_abfree[k % kAS]);
        PH(2);
      }
      if (t == 0) PH_DUMP(16);
    }
  } else if (warp < kE) {
    // ------------------------------------------------------------ expansion warps (thread = row = TMEM lane)
    // per unit: B (z of the group for NT tokens), A (this row's planes as bytes 0/1 -> TMEM), the row's
    // coefficients c_t and the tokens' scales for the epilogue warps; then A/B ready -> the issuers
    asm volatile("griddepcontrol.wait;" ::: "memory");   // activations from here on
    PH_DECL
    const int lq = warp & 3, sub = warp >> 2;       // lane quarter; the plane this warp expands
    const int r = 32 * lq + lane;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int swz = chunk_swizzle(K, r);
    const int bn = tid >> 2, bq = tid & 3;         // B-build job: token bn, 32-element chunk bq
    const bool bwarp = warp * 8 < NT;             // warp-uniform: this warp has B-build jobs
    uint32_t X[8];
    float sxn = 0.f;
    auto load_x = [&](int g) {
      if (bwarp) {
        const bool live = bn < p.ntok;
        const uint32_t* src = p.xplanes + ((size_t)bn * NG + g) * p.l * 4 + bq;
#pragma unroll
        for (int j = 0; j < 8; ++j) X[j] = live ? __ldg(src + min(j, p.l - 1) * 4) : 0u;
        sxn = (!DEBUG && live && bq == 0) ? __ldg(p.xscales + (size_t)bn * NG + g) : 0.f;
      }
    };
    load_x(V0 % NG);
    int rb = V0 / NG, g = V0 - (V0 / NG) * NG;
    for (int k = 0; k < n; ++k) {
      const int rows = rows_of(rb);
      if (k >= kAS) ZT_WAIT_CRIT(&bar_abfree[k % kAS], ((k - kAS) / kAS) & 1);   // slot read by MMA(k - kAS)
      PH(0);
      if (bwarp && !(ZT_ABL & 1)) {
        uint32_t Z[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) Z[j] = X[j];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const uint32_t x = ((Z[j] >> 1) ^ Z[j + 1]) & 0x55555555u;
          Z[j + 1] ^= x;
          Z[j] ^= x << 1;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (!(j & 2)) {
            const uint32_t x = ((Z[j] >> 2) ^ Z[j + 2]) & 0x33333333u;
            Z[j + 2] ^= x;
            Z[j] ^= x << 2;
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = ((Z[j] >> 4) ^ Z[j + 4]) & 0x0F0F0F0Fu;
          Z[j + 4] ^= x;
          Z[j] ^= x << 4;
        }
        // register s, byte i = z(32 bq + 8 i + s) = k-order byte 4 s + i of B row bn (MMA q = bq)
        uint8_t* row = sB + (k % kAS) * kBBytes + bq * (NT * 32) + (bn >> 3) * 256 + (bn & 7) * 16;
        *reinterpret_cast<uint4*>(row) = make_uint4(Z[0], Z[1], Z[2], Z[3]);
        *reinterpret_cast<uint4*>(row + 128) = make_uint4(Z[4], Z[5], Z[6], Z[7]);
        if (bq == 0) s_sx[k % kRing][bn] = sxn;
      }
      const int g_next = g + 1 == NG ? 0 : g + 1;
      if (k + 1 < n && !(ZT_ABL & 8)) load_x(g_next);
      PH(1);
      const int slot = k % kSlots;
      mbar_wait(&bar_full[slot], (k / kSlots) & 1);
      PH(2);
      const uint8_t* sl = ring + slot * kSlotBytes;
      if (sub < K && !(ZT_ABL & 2)) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(sl + r * 16 * K + 16 * (sub ^ swz));
        const uint32_t wq[4] = {w4.x, w4.y, w4.z, w4.w};
        uint32_t a[32];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int s = 0; s < 8; ++s) a[8 * q + s] = shr_fma(wq[q], s) & 0x01010101u;
        tmem_st32(tmem + lane_base + 32 * (kAS * sub + k % kAS), a);
      }
      if (sub == K - 1) {                            // c_t = s r^t + b (Eq. 4) of this row, for the epilogue
        uint32_t sbw = 0, ri = 0;
        if (r < rows) {
          sbw = *reinterpret_cast<const uint32_t*>(sl + rows * 16 * K + 4 * r);
          ri = sl[rows * (16 * K + 4) + r];
        }
        const float s_ = __half2float(__ushort_as_half((unsigned short)(sbw & 0xffffu)));
        const float b_ = __half2float(__ushort_as_half((unsigned short)(sbw >> 16)));
#pragma unroll
        for (int t = 0; t < K; ++t) s_c[((k % kRing) * K + t) * 128 + r] = fmaf(s_, s_rpow[ri * K + t], b_);
      }
      PH(3);
      tmem_wait_st();
      fence_proxy_async();              // B (generic stores) -> the MMA (async proxy); slot reads -> the refill
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar_a[k % kAS]);
        // the last expansion warp done with this slot refills it with unit k + kSlots
        if (atomicAdd(&s_rel[slot], 1u) == kE - 1) {
          s_rel[slot] = 0;
          if (k + kSlots < n) {
            mbar_expect_tx(&bar_full[slot], unit_bytes(V0 + k + kSlots));
            bulk_g2s(ring + slot * kSlotBytes, unit_src(V0 + k + kSlots), unit_bytes(V0 + k + kSlots), &bar_full[slot]);
          }
        }
      }
      PH(4);
      g = g_next;
      if (g == 0) ++rb;
    }
    if (warp == 0) PH_DUMP(0);
  } else {
    // ------------------------------------------------------------ epilogue warps (thread = row = TMEM lane)
    asm volatile("griddepcontrol.wait;" ::: "memory");   // workspace and Y from here on
    PH_DECL
    const int ew = warp - kE;
    const int lq = warp & 3, th = ew >> 2;           // lane quarter; token half
    const int r = 32 * lq + lane;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int etid = ew * 32 + lane;                  // 0 .. 255
    float y[TQ];
#pragma unroll
    for (int i = 0; i < TQ; ++i) y[i] = 0.f;

    // leaving row block rb: write y (or hand the CTA partial to the last-arriving CTA of rb)
    auto flush = [&](int rb, int rows) {
      const bool shared = (long)rb * NG < V0 || (long)(rb + 1) * NG > V1;
      if (!shared) {
        if (!DEBUG && r < rows)
#pragma unroll
          for (int i = 0; i < TQ; ++i) {
            const int tok = th * TQ + i;
            if (tok < p.ntok) p.Y[(size_t)tok * p.M + (size_t)rb * 128 + r] = y[i];
          }
      } else if (!DEBUG) {
        const int myslot = rb == V0 / NG ? 0 : 1;
        float* part = p.ws_part + ((size_t)cta * 2 + myslot) * (NT * 128);
#pragma unroll
        for (int i = 0; i < TQ; ++i) __stcg(part + (th * TQ + i) * 128 + r, y[i]);
        named_bar(1, kP * 32);
        if (etid == 0) s_old = atomicAdd(p.ws_cnt + rb, 1u);
        named_bar(1, kP * 32);
        const int c0 = unit_cta(rb * NG, p.qq, p.rr), c1 = unit_cta((rb + 1) * NG - 1, p.qq, p.rr);
        // at rest the counter is 0xFFFFFFFF: the k-th arrival reads k - 2 (mod 2^32)
        if (s_old + 2u == (unsigned int)(c1 - c0 + 1)) {
          float sum[TQ];
#pragma unroll
          for (int i = 0; i < TQ; ++i) sum[i] = 0.f;
          for (int cc = c0; cc <= c1; ++cc) {
            const int sl = rb == range_begin(cc, p.qq, p.rr) / NG ? 0 : 1;
            float* src = p.ws_part + ((size_t)cc * 2 + sl) * (NT * 128);
            if (cc == cta) {
#pragma unroll
              for (int i = 0; i < TQ; ++i) sum[i] += y[i];
              continue;
            }
            // all TQ words of the slot in one batch (one L2 round trip), reloaded while any is the sentinel
            uint32_t w[TQ];
            for (long spins = 0;; ++spins) {
              bool miss = false;
#pragma unroll
              for (int i = 0; i < TQ; ++i) {
                w[i] = ld_relaxed_u32(src + (th * TQ + i) * 128 + r);
                miss |= w[i] == kSentinel;
              }
              if (!miss) break;
              if (spins > (1L << 26)) __trap();          // stores already issued never landed
            }
#pragma unroll
            for (int i = 0; i < TQ; ++i) sum[i] += __uint_as_float(w[i]);
          }
          for (int cc = c0; cc <= c1; ++cc) {
            const int sl = rb == range_begin(cc, p.qq, p.rr) / NG ? 0 : 1;
            unsigned int* dst = reinterpret_cast<unsigned int*>(p.ws_part) + ((size_t)cc * 2 + sl) * (NT * 128);
#pragma unroll
            for (int i = 0; i < TQ; ++i) dst[(th * TQ + i) * 128 + r] = kSentinel;
          }
          if (etid == 0) p.ws_cnt[rb] = kSentinel;
          if (r < rows)
#pragma unroll
            for (int i = 0; i < TQ; ++i) {
              const int tok = th * TQ + i;
              if (tok < p.ntok) p.Y[(size_t)tok * p.M + (size_t)rb * 128 + r] = sum[i];
            }
        }
      }
#pragma unroll
      for (int i = 0; i < TQ; ++i) y[i] = 0.f;
    };

    int rb = V0 / NG, g = V0 - (V0 / NG) * NG, rb_cur = rb;
    for (int k = 0; k < n; ++k) {
      const int rows = rows_of(rb);
      if (rb != rb_cur) {
        PH(6);
        flush(rb_cur, rows_of(rb_cur));
        PH(7);
        rb_cur = rb;
      }
      const int db = k % kDBuf;
      PH(6);
#pragma unroll
      for (int t = 0; t < K; ++t) mbar_wait_backoff(&bar_dfull[t][db], (k / kDBuf) & 1);
      tc_fence_after();
      PH(4);
      // token chunks of TC columns: all K planes of a chunk are loaded before one tcgen05.wait::ld
#pragma unroll
      for (int c0 = 0; c0 < TQ; c0 += TC) {
        uint32_t v[K][TC];
#pragma unroll
        for (int t = 0; t < K; ++t) tmem_ld<TC>(tmem + lane_base + kDCol + NT * (t + K * db) + th * TQ + c0, v[t]);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < K; ++t) pin<TC>(v[t]);
        if (c0 + TC == TQ) {                           // D of this unit fully read: the issuers may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane < K) mbar_arrive(&bar_dempty[lane][db]);
        }
        if (DEBUG) {
          if (r < rows)
#pragma unroll
            for (int t = 0; t < K; ++t)
#pragma unroll
              for (int i = 0; i < TC; ++i) {
                const int tok = th * TQ + c0 + i;
                if (tok < p.ntok) p.Tdbg[(((size_t)(rb * 128 + r) * NG + g) * K + t) * p.ntok + tok] = (int32_t)v[t][i];
              }
        } else {
          float acc[TC];
#pragma unroll
          for (int t = 0; t < K; ++t) {
            const float c = s_c[((k % kRing) * K + t) * 128 + r];
#pragma unroll
            for (int i = 0; i < TC; ++i)
              acc[i] = t == 0 ? c * __int2float_rn((int)v[t][i]) : fmaf(c, __int2float_rn((int)v[t][i]), acc[i]);
          }
#pragma unroll
          for (int i = 0; i < TC; ++i) y[c0 + i] = fmaf(s_sx[k % kRing][th * TQ + c0 + i], acc[i], y[c0 + i]);
        }
      }
      PH(5);
      g = g + 1 == NG ? 0 : g + 1;
      if (g == 0) ++rb;
    }
    PH(6);
    if (n > 0) flush(rb_cur, rows_of(rb_cur));
    PH(7);
    if (ew == 0) PH_DUMP(8);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side
static int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

struct Plan {
  int NG, n_full, tail_rows, n_rb, Us, C;
};
static Plan make_plan(const sbvr_weights* w) {
  Plan pl;
  pl.NG = w->N / kG;
  pl.n_full = w->M / kRowBlock;
  pl.tail_rows = w->M % kRowBlock;
  pl.n_rb = pl.n_full + (pl.tail_rows ? 1 : 0);
  pl.Us = pl.n_rb * pl.NG;
  // at least ZT_MIN_UNITS units per CTA: a row block split over fewer CTAs has fewer partials to combine (the
  // last-arriving CTA reads one slot per contributor), which dominates small matrices at large T
  const int by_units = (pl.Us + ZT_MIN_UNITS - 1) / ZT_MIN_UNITS;
  pl.C = num_sms() < by_units ? num_sms() : (by_units < 1 ? 1 : by_units);
  return pl;
}

static int nt_for(int ntok) { return ntok <= 8 ? 8 : ntok <= 16 ? 16 : 32; }
static size_t cnt_bytes(const Plan& pl) { return ((size_t)(pl.n_rb + 1) * 4 + 255) / 256 * 256; }

template <int K, int NT, bool DEBUG>
static cudaError_t launch_one(const ZtParams& p, int C, cudaStream_t st) {
  const int smem = kSlots * ((128 * (16 * K + 5) + 127) / 128 * 128) + kAS * 4 * NT * 32 + kRing * K * 128 * 4;
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemv_zt_kernel<K, NT, DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemv_zt_kernel<K, NT, DEBUG>, p);
}

template <int K>
static cudaError_t launch_k(const ZtParams& p, int C, int NT, bool debug, cudaStream_t st) {
  if (debug) {
    switch (NT) {
      case 8: return launch_one<K, 8, true>(p, C, st);
      case 16: return launch_one<K, 16, true>(p, C, st);
      default: return launch_one<K, 32, true>(p, C, st);
    }
  }
  switch (NT) {
    case 8: return launch_one<K, 8, false>(p, C, st);
    case 16: return launch_one<K, 16, false>(p, C, st);
    default: return launch_one<K, 32, false>(p, C, st);
  }
}

}  // namespace zt

bool zt_supported(const sbvr_weights* w, const sbvr_act* x) {
  return x->kind == SBVR_ACT_SBVR && w->K >= 1 && w->K <= zt::kMaxPlanes;
}

size_t zt_workspace_bytes(const sbvr_weights* w, int T) {
  const zt::Plan pl = zt::make_plan(w);
  const int NT = zt::nt_for(T < zt::kMaxNT ? T : zt::kMaxNT);
  return zt::cnt_bytes(pl) + (size_t)pl.C * 2 * NT * 128 * sizeof(float);
}

sbvr_status launch_gemv_zt(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                           int32_t* T_debug, cudaStream_t st) {
  using namespace zt;
  if (!zt_supported(w, x)) return set_error(SBVR_ERR_UNSUPPORTED, "ZT: SBVR-x and K <= 4 only (K=%d)", w->K);
  const Plan pl = make_plan(w);
  const bool debug = T_debug != nullptr;
  if (!debug && (!ws || ws_bytes < zt_workspace_bytes(w, T)))
    return set_error(SBVR_ERR_WORKSPACE, "ZT: workspace %zu bytes < required %zu", ws_bytes, zt_workspace_bytes(w, T));
  ZtParams p;
  p.units = w->data;
  p.ratio_pow = w->ratio_pow;
  p.M = w->M; p.N = w->N; p.l = x->l; p.n_ratio = w->n_ratio;
  p.n_full = pl.n_full;
  p.tail_rows = pl.tail_rows;
  p.Us = pl.Us;
  p.qq = pl.Us / pl.C;
  p.rr = pl.Us % pl.C;
  p.ws_cnt = ws ? reinterpret_cast<unsigned int*>(ws) : nullptr;
  p.ws_part = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + cnt_bytes(pl)) : nullptr;
  p.Tdbg = T_debug;
  {
    const char* tsp = getenv("SBVR_TS_PTR");
    p.ts = tsp ? reinterpret_cast<unsigned long long*>(strtoull(tsp, nullptr, 0)) : nullptr;
  }
  const uint32_t* xp = static_cast<const uint32_t*>(x->data);
  for (int done = 0; done < T; done += kMaxNT) {
    const int ntok = T - done < kMaxNT ? T - done : kMaxNT;
    p.ntok = ntok;
    p.xplanes = xp + (size_t)done * pl.NG * x->l * 4;
    p.xscales = x->scales + (size_t)done * pl.NG;
    p.Y = Y ? Y + (size_t)done * w->M : nullptr;
    const int NT = nt_for(ntok);
    cudaError_t e;
    switch (w->K) {
      case 1: e = launch_k<1>(p, pl.C, NT, debug, st); break;
      case 2: e = launch_k<2>(p, pl.C, NT, debug, st); break;
      case 3: e = launch_k<3>(p, pl.C, NT, debug, st); break;
      default: e = launch_k<4>(p, pl.C, NT, debug, st); break;
    }
    if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "gemv_zt setup: %s", cudaGetErrorString(e));
    sbvr_status s = check_launch("gemv_zt_kernel");
    if (s != SBVR_OK) return s;
    if (debug) break;
  }
  return SBVR_OK;
}

}  // namespace sbvr
