// gemv_group.cu -- grouped SBVR GEMV: several independent batch-1 GEMVs y_p = W_p x_p (§4.4, P:245-251;
// SBVR-x, the AND+popcount form of gemv_mma.cuh) in ONE persistent launch (sbvr_gemv_group, include/sbvr.h).
//
// Why: a batch-1 GEMV of a decoder layer moves 2-32 MB, so a launch that streams it at the core rate lasts only
// 3-20 us, and every launch pays a fixed cost that does not shrink with the matrix -- first bytes ~2 us after the
// CTA starts, split-K combine, CTA tail spread, the next launch's griddepcontrol.wait (~45% of the 4-launch step,
// DESIGN.md §7).  Here the problems' unit records are concatenated into one global work sequence
//     problem 0's units (row-block-major, as in HBM) | problem 1's units | ...
// split into balanced contiguous CTA ranges; the fixed costs are paid once per group, not once per matrix, and a
// ring runs on across matrix boundaries (the next matrix's first records are in flight while one is finishing).
//
// Work unit = one whole unit record (128 rows x 1 group, contiguous in HBM: sbvr.h), fetched by ONE
// cp.async.bulk into a slot shared by a PAIR of warps: warp 2q computes rows 0-63 of it, warp 2q+1 rows 64-127.
// A pair walks a contiguous range of units (consecutive units of a matrix are consecutive records: the copy source
// just advances by one record).  Both warps wait on the slot's full barrier; each releases it with a shared-memory
// counter and the SECOND releaser refills it -- nobody waits for the partner.  (Per-warp 64-row rings, as in
// gemv_mma, need three copies per unit -- planes, scale/bias, ratio indices of a half record -- and a per-unit
// address computation executed by the whole warp: ~45% of the instructions of the first group kernel were such
// per-unit overhead, ncu source page, profiles/r02_group_ncu.md.)
//
// Arithmetic per (row, group) is the MMA kernel's, bit for bit: A = plane word & (0x01010101 << s), B = activation
// plane j bit-sliced x 2^(7-s), mma.m16n8k32.u8 accumulates 128 P_tj, epilogue u = D0 + kappa D1, exact int->float,
// Horner over t in fp32x2, y += s_x (s sum_t r^t u_t + b sum_t u_t).  A band (64 rows: one half of a row block of one
// matrix) shared by several warps / CTAs is combined by the deterministic last-arriver reduction of gemv_mma.cuh
// (smem counter, sum in warp order; global counter + sentinel-validated slots, sum in CTA order).  Restrictions
// (checked by the ABI): T = 1, SBVR-x, SBVR_META_GROUP, K in 2..4 and the same for every problem, M % 128 == 0,
// 1..8 problems.
#include "gemv_mma.cuh"

namespace sbvr {
namespace grp {
using namespace mma;

constexpr int kMaxProb = SBVR_GROUP_MAX;
constexpr int kMaxPeers = 8;
#ifndef SBVR_GROUP_WARPS
#define SBVR_GROUP_WARPS 8
#endif
#ifndef SBVR_GROUP_CTAS
#define SBVR_GROUP_CTAS 2
#endif
#ifndef SBVR_GROUP_SLOTS
#define SBVR_GROUP_SLOTS 2
#endif
constexpr int kGW = SBVR_GROUP_WARPS;     // warps per CTA (even: warp pairs)
constexpr int kGC = SBVR_GROUP_CTAS;      // resident CTAs per SM
constexpr int kGS = SBVR_GROUP_SLOTS;     // ring slots per warp pair
constexpr int kPairs = kGW / 2;
static_assert(kGW % 2 == 0, "warp pairs");

template <int K>
struct UnitGeom {
  static constexpr int kBytes = 128 * (16 * K + 5);            // one unit record (sbvr.h)
  static constexpr int kSlot = (kBytes + 127) / 128 * 128;
  static constexpr int kSb = 128 * 16 * K;                     // offset of the scale/bias words
  static constexpr int kRi = 128 * (16 * K + 4);               // offset of the ratio-index bytes
  static constexpr int kSmem = kPairs * kGS * kSlot + kGW * 2 * 64 * 4;
};

struct GProb {
  const uint8_t* units;     // unit records of W_p (full 128-row blocks)
  const uint32_t* xplanes;  // [NG][l][4]
  const float* xscales;     // [NG]
  float* Y[kMaxPeers];      // [M] -- or, fused all-gather (sbvr_gemv_group_to_peers), every rank's full y at this
                            // rank's row offset (ny pointers)
  int NG;                   // groups per row
  int rbbase;               // first global row block of this problem
  int ubase;                // first global unit of this problem
};

struct GroupParams {
  GProb pr[kMaxProb];
  const float* ratio_pow[kMaxProb];   // [n_ratio][K] per problem
  int n_ratio[kMaxProb];
  int np;                   // problems
  int ny;                   // y destinations per problem (1; n_peers for the fused all-gather)
  int Us;                   // total units
  int C, qq, rr;            // CTAs and the unit partition over CTAs
  int l, one;
  float* ws_part;           // [CTA][4][64] fp32 partials: (first / last row block of the CTA) x (half) (kSentinel at rest)
  unsigned int* ws_cnt;     // [global band = 2 * global row block + half] arrival counters (0xFFFFFFFF at rest)
  unsigned long long* ts;   // -DSBVR_DIAG only (env SBVR_TS_PTR): [CTA][warp][8] stamps 0-2, smid, units
  // SBVR_ACT_FP16_Q problems: x converted in the kernel (Eq. 12, the arithmetic of encode_vector_kernel)
  int conv;                 // 1: every problem's x is fp16, converted in the prologue
  const uint16_t* xh[kMaxProb];   // fp16 x of each problem
  int gbase[kMaxProb];      // first global x-group of each problem
  int n_xg;                 // x-groups of all problems
  uint32_t* xq_planes;      // workspace: [x-group][l][4] converted planes (pr[].xplanes point here)
  float* xq_scales;         // workspace: [x-group] s_x
  unsigned int* conv_cnt;   // workspace: converted x-groups (0xFFFFFFFF at rest)
  unsigned int* exit_cnt;   // workspace: CTAs finished (0xFFFFFFFF at rest)
};
#ifdef SBVR_DIAG
__device__ int getenv_diag_tma = 1;
#define GTSW(slot) do { if (P.ts && lane == 0) P.ts[((size_t)blockIdx.x * kGW + wib) * 16 + (slot)] = gtime(); } while (0)
#else
#define GTSW(slot) do { } while (0)
#endif

__device__ __forceinline__ int prob_of(const GroupParams& P, int u, int p = 0) {
#pragma unroll 1
  while (p + 1 < P.np && u >= P.pr[p + 1].ubase) ++p;
  return p;
}
// global row block of global unit u
__device__ __forceinline__ int rb_of(const GroupParams& P, int u) {
  const int p = prob_of(P, u);
  return P.pr[p].rbbase + (u - P.pr[p].ubase) / P.pr[p].NG;
}

#ifdef SBVR_GROUP_X_RELAXED
__device__ __forceinline__ uint32_t ldx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ldx(const float* p) { return __uint_as_float(ldx(reinterpret_cast<const uint32_t*>(p))); }
#else
__device__ __forceinline__ uint32_t ldx(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ float ldx(const float* p) { return __ldcg(p); }
#endif

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Eq. 12 for one group of 128 fp16 values by one warp, bit-identical to encode_vector_kernel (the same fp32 IEEE
// operations): s_x = absmax / (2^(l-1) - 1) (__fdiv_rn), z = clamp(rne(x / s_x)), l-bit two's-complement planes
// by ballot; word (plane j, 32-element word c) -> planes[4 j + c], s_x -> *scale.
__device__ __forceinline__ void convert_group(const GroupParams& P, const uint16_t* xg, uint32_t* planes, float* scale) {
  const int lane = threadIdx.x & 31;
  float v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = __half2float(__ushort_as_half(xg[32 * c + lane]));
  float a = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
  const int zmax = (1 << (P.l - 1)) - 1;
  const float sx = (a != 0.0f) ? __fdiv_rn(a, (float)zmax) : 0.0f;
  const uint32_t lmask = (1u << P.l) - 1u;
  uint32_t mine = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    int z = 0;
    if (sx != 0.0f) {
      z = __float2int_rn(__fdiv_rn(v[c], sx));
      z = min(max(z, -zmax), zmax);
    }
    const uint32_t u = (uint32_t)z & lmask;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t word = __ballot_sync(0xffffffffu, (u >> j) & 1u);
      if (lane == 4 * j + c) mine = word;
    }
  }
#ifdef SBVR_GROUP_CONV_PLAIN_ST
  if (lane < 4 * P.l) planes[lane] = mine;
  if (lane == 0) *scale = sx;
#else
  if (lane < 4 * P.l) __stcg(planes + lane, mine);
  if (lane == 0) __stcg(scale, sx);
#endif
}

template <int K>
__device__ __forceinline__ void issue_unit_rec(uint8_t* slot, uint64_t* bar, const GroupParams& P, int u, int p_hint) {
  using UG = UnitGeom<K>;
  const int p = prob_of(P, u, p_hint);
  const uint8_t* src = P.pr[p].units + (size_t)(u - P.pr[p].ubase) * UG::kBytes;
  mbar_expect_tx(bar, UG::kBytes);
  bulk_g2s(slot, src, UG::kBytes, bar);
}

template <int K>
__global__ void __launch_bounds__(kGW * 32, kGC) gemv_group_kernel(GroupParams P) {
  using UG = UnitGeom<K>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float s_rat[kMaxProb * 64];          // r_i of every problem (Horner of sum_t r^t u_t)
  __shared__ uint64_t s_full[kPairs][kGS];        // slot filled (tx bytes)
  __shared__ unsigned int s_rel[kPairs][kGS];     // warps of the pair done with the slot's unit
  __shared__ unsigned int s_cnt[2 * kGW];         // warps done with a band, by (first holder, its first/last band)
  __shared__ int s_fb[kGW];                       // first global band of each warp
  __shared__ int s_lb[kGW];                       // last global band of each warp (-1: no units)
  float* s_part = reinterpret_cast<float*>(smem + kPairs * kGS * UG::kSlot);   // [warps][2][64]
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int pair = wib >> 1, hf = wib & 1;        // warp pair and the half (rows 64 hf .. 64 hf + 63) it computes
  GTSW(0);
  const int cta = blockIdx.x;
  const int V0 = cta * P.qq + min(cta, P.rr);
  const int V1 = V0 + P.qq + (cta < P.rr ? 1 : 0);
  // this CTA's units split over its warp pairs: pair q takes units [U0, U0 + n)
  const int nU = V1 - V0;
  const int pq = nU / kPairs, pr = nU % kPairs;
  const int U0 = V0 + pair * pq + min(pair, pr);
  const int n = pq + (pair < pr ? 1 : 0);
  uint8_t* ring = smem + pair * kGS * UG::kSlot;
  if (hf == 0 && lane == 0 && n > 0) {
    // weights are immutable: their copies start before we wait for the previous kernel
#pragma unroll
    for (int s2 = 0; s2 < kGS; ++s2) {
      mbar_init(&s_full[pair][s2], 1);
      s_rel[pair][s2] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int p0 = prob_of(P, U0);
#pragma unroll
    for (int s2 = 0; s2 < kGS; ++s2)
      if (s2 < n) issue_unit_rec<K>(ring + s2 * UG::kSlot, &s_full[pair][s2], P, U0 + s2, p0);
#ifdef SBVR_DIAG
    if (P.ts && getenv_diag_tma) {            // diagnostics: when does the first prefetched record land?
      mbar_wait(&s_full[pair][0], 0);
      P.ts[((size_t)blockIdx.x * kGW + wib) * 16 + 7] = gtime();
    }
#endif
  }
  for (int i = threadIdx.x; i < kMaxProb * 64; i += blockDim.x) {
    const int pp = i >> 6, ri = i & 63;
    s_rat[i] = (pp < P.np && ri < P.n_ratio[pp] && K >= 2) ? P.ratio_pow[pp][ri * K + 1] : 0.f;
  }
  for (int i = threadIdx.x; i < 2 * kGW; i += blockDim.x) s_cnt[i] = 0u;
  if (threadIdx.x < kGW) {
    const int w2 = threadIdx.x, q2 = w2 >> 1;
    const int u0 = V0 + q2 * pq + min(q2, pr), n2 = pq + (q2 < pr ? 1 : 0);
    s_fb[w2] = n2 > 0 ? 2 * rb_of(P, u0) + (w2 & 1) : 0x7fffffff;
    s_lb[w2] = n2 > 0 ? 2 * rb_of(P, u0 + n2 - 1) + (w2 & 1) : -1;
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");   // activations / workspace / y from here
  GTSW(3);
  if (P.conv) {
    // SBVR_ACT_FP16_Q: Eq. 12 conversion of every problem's fp16 x, distributed over the grid (warp w of CTA c
    // converts x-groups w * C + c, w * C + c + kGW * C, ...: the first warps of many SMs), planes and scales to the
    // workspace, then a grid-wide arrival count; every warp waits for it before its first x load (below).
    for (int q = wib * P.C + cta; q < P.n_xg; q += kGW * P.C) {
      int pp = 0;
      while (pp + 1 < P.np && q >= P.gbase[pp + 1]) ++pp;
      convert_group(P, P.xh[pp] + (size_t)(q - P.gbase[pp]) * kG, P.xq_planes + (size_t)q * 4 * P.l, P.xq_scales + q);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAdd(P.conv_cnt, 1u);
      }
    }
  }
  if (P.conv) {
    // all x-groups converted: one thread per CTA polls (acquire), the CTA barrier orders everyone's x loads after
    // it (the counter rests at 0xFFFFFFFF: after k arrivals it reads k - 1)
    if (threadIdx.x == 0)
      for (unsigned int v = ld_acquire_u32(P.conv_cnt); v + 1u < (unsigned int)P.n_xg || v == kSentinel;
           v = ld_acquire_u32(P.conv_cnt))
        __nanosleep(64);
    __syncthreads();
    GTSW(6);
  }
  if (n > 0) {

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
    // lane (gq, c) reads word c of rows 16 i + gq and 16 i + gq + 8, i = 4 hf .. 4 hf + 3 (chunk swizzle of sbvr.h)
    const int swz_a = chunk_swizzle(K, gq);         // (= chunk_swizzle(K, gq + 8) for K = 2, 3, 4)
    const int row_a = 64 * hf + gq;                 // + 16 i' (i' = 0..3), + 8 for the second row of the lane
    // lane-constant byte offsets of word c of plane t in the lane's first row (the swizzle folded in once): every
    // plane-word load of a unit is then slot base + lo[t] + an immediate
    uint32_t lo[K];
#pragma unroll
    for (int t = 0; t < K; ++t) lo[t] = (uint32_t)(row_a * 16 * K + 4 * c + 16 * (t ^ swz_a));

    float2 acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
    auto store_y = [&](int pp, int off, float v) {  // y row (local to problem pp) -> its destination(s)
#pragma unroll 1
      for (int j = 0; j < P.ny; ++j) P.pr[pp].Y[j][off] = v;
    };

    // position of the current unit: problem p, global row block rb, group g (+ the problem's constants)
    int p = prob_of(P, U0);
    int NGp = P.pr[p].NG, rbb = P.pr[p].rbbase;
    int rb = rbb + (U0 - P.pr[p].ubase) / NGp, g = (U0 - P.pr[p].ubase) % NGp;
    int rb_end = p + 1 < P.np ? P.pr[p + 1].rbbase : 0x7fffffff;
    const uint32_t* xpl = P.pr[p].xplanes;
    const float* xsc = P.pr[p].xscales;
    int rat_off = p * 64;
    int slot = 0;
    uint32_t phase = 0;
    uint32_t Xn = ldx(xpl + (size_t)g * xstride + xoff);   // (L2: FP16_Q planes are written by this kernel)
    float sxn = ldx(xsc + g);
#ifdef SBVR_DIAG
    if (P.ts && lane == 0 && (Xn ^ __float_as_uint(sxn)) != 0x9E3779B9u) GTSW(8);   // first x landed
#endif

    for (int k = 0; k < n; ++k) {
      // ---- B operand for group g: activation plane gq, word c, bit-sliced and pre-scaled by 2^(7-s)
      uint32_t Bq[4][2];
      const float sx = sxn;
      {
        const uint32_t X = Xn & xmask;
  #pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          Bq[q2][0] = bslice(X, 2 * q2);
          Bq[q2][1] = bslice(X, 2 * q2 + 1);
        }
      }
      const int cur_p = p, cur_rb = rb, cur_rat = rat_off;
      const int ycur = 128 * (rb - rbb) + 64 * hf;    // this warp's first y row of the unit's band
      const int ub0 = P.pr[p].ubase + (rb - rbb) * NGp;           // the row block's first and end global units
      const int ub1 = ub0 + NGp;
      // advance to the next unit (problem switch: reload the problem's constants)
      if (++g == NGp) {
        g = 0;
        if (++rb == rb_end) {
          ++p;
          NGp = P.pr[p].NG;
          rbb = P.pr[p].rbbase;
          rb_end = p + 1 < P.np ? P.pr[p + 1].rbbase : 0x7fffffff;
          xpl = P.pr[p].xplanes;
          xsc = P.pr[p].xscales;
          rat_off = p * 64;
        }
      }
      const bool has_next = k + 1 < n;
      if (has_next) {
        Xn = ldx(xpl + (size_t)g * xstride + xoff);
        sxn = ldx(xsc + g);
      }

      uint8_t* sl = ring + slot * UG::kSlot;
      mbar_wait(&s_full[pair][slot], phase);
      if (k == 0) GTSW(1);

  #pragma unroll
      for (int ib = 0; ib < 4; ib += 2) {
        uint32_t w[2][2 * K];
        uint32_t sb0[2], sb1[2];
        float2 r2[2];
  #pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = row_a + 16 * (ib + j);
  #pragma unroll
          for (int t = 0; t < K; ++t) {
            const uint8_t* pa = sl + lo[t] + 16 * (ib + j) * 16 * K;
            w[j][2 * t] = *reinterpret_cast<const uint32_t*>(pa);
            w[j][2 * t + 1] = *reinterpret_cast<const uint32_t*>(pa + 8 * 16 * K);
          }
          sb0[j] = *reinterpret_cast<const uint32_t*>(sl + UG::kSb + 4 * r);
          sb1[j] = *reinterpret_cast<const uint32_t*>(sl + UG::kSb + 4 * (r + 8));
          r2[j] = make_float2(s_rat[cur_rat + sl[UG::kRi + r]], s_rat[cur_rat + sl[UG::kRi + r + 8]]);
        }
        // ---- AND + popcount on the tensor pipe: 2 x K independent chains (tile, plane) of 4 MMAs
        int D[2][K][4];
  #pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          const uint32_t m0 = 0x01010101u << (2 * q2), m1 = 0x01010101u << (2 * q2 + 1);
  #pragma unroll
          for (int t = 0; t < K; ++t)
  #pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint32_t a0 = w[j][2 * t] & m0, a1 = w[j][2 * t + 1] & m0;
              const uint32_t a2 = w[j][2 * t] & m1, a3 = w[j][2 * t + 1] & m1;
              if (q2 == 0)
                mma_u8(D[j][t], a0, a1, a2, a3, Bq[q2][0], Bq[q2][1], 0, 0, 0, 0);
              else
                mma_u8(D[j][t], a0, a1, a2, a3, Bq[q2][0], Bq[q2][1], D[j][t][0], D[j][t][1], D[j][t][2], D[j][t][3]);
            }
        }
  #pragma unroll
        for (int j = 0; j < 2; ++j) {
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
          acc[ib + j] = __ffma2_rn(make_float2(sx, sx), v, acc[ib + j]);
        }
      }

      // ---- release the slot; the second warp of the pair to release it refills it with unit k + kGS
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&s_rel[pair][slot], 1u) == 1u) {
          s_rel[pair][slot] = 0u;
          if (k + kGS < n) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_unit_rec<K>(sl, &s_full[pair][slot], P, U0 + k + kGS, cur_p);
          }
        }
      }
      if (++slot == kGS) { slot = 0; phase ^= 1u; }

      // ---- leaving band (cur_rb, hf): warp-level then CTA-level combine (see gemv_mma.cuh)
      if (!has_next || rb != cur_rb) {
        const int b = 2 * cur_rb + hf;
        // warps of this CTA holding band b: same half, band within their range (a set of warps of one parity)
        const unsigned int holders =
            __ballot_sync(0xffffffffu, lane < kGW && (lane & 1) == hf && s_fb[min(lane, kGW - 1)] <= b &&
                                           s_lb[min(lane, kGW - 1)] >= b);
        const int wf = __ffs(holders) - 1, nh = __popc(holders);
        const bool shared = V0 > ub0 || V1 < ub1;                 // other CTAs hold units of the row block
        float* sp = s_part + ((size_t)wib * 2 + (b == s_fb[wib] ? 0 : 1)) * 64;
  #pragma unroll
        for (int i = 0; i < 4; ++i) {
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
        if (nh > 1) {
          __syncwarp();
          unsigned int old = 0;
          if (lane == 0) {
            __threadfence_block();
            old = atomicAdd(&s_cnt[wf * 2 + (b == s_fb[wf] ? 0 : 1)], 1u);
          }
          old = __shfl_sync(0xffffffffu, old, 0);
          last = old == (unsigned int)(nh - 1);
        }
        if (last) {
          __syncwarp();
          __threadfence_block();
          float v[2];
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            float sum = 0.f;
            for (unsigned int m = holders; m; m &= m - 1) {       // contributing warps, in warp order
              const int w2 = __ffs(m) - 1;
              sum += s_part[((size_t)w2 * 2 + (b == s_fb[w2] ? 0 : 1)) * 64 + lane + 32 * h];
            }
            v[h] = sum;
          }
          if (!shared) {
  #pragma unroll
            for (int h = 0; h < 2; ++h) store_y(cur_p, ycur + lane + 32 * h, v[h]);
          } else {
            // last-arriver reduction over the CTAs holding units of the row block (deterministic CTA order; nobody
            // waits on another CTA's progress: see gemv_mma.cuh)
            const int myslot = (V0 >= ub0 ? 0 : 2) + hf;
            float* part = P.ws_part + ((size_t)cta * 4 + myslot) * 64;
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
                    const float* src = P.ws_part + ((size_t)cc * 4 + (v0c >= ub0 ? 0 : 2) + hf) * 64;
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
                unsigned int* dst =
                    reinterpret_cast<unsigned int*>(P.ws_part) + ((size_t)cc * 4 + (v0c >= ub0 ? 0 : 2) + hf) * 64;
  #pragma unroll
                for (int h = 0; h < 2; ++h) dst[lane + 32 * h] = kSentinel;
              }
              if (lane == 0) P.ws_cnt[b] = kSentinel;
  #pragma unroll
              for (int h = 0; h < 2; ++h) store_y(cur_p, ycur + lane + 32 * h, sum[h]);
            }
          }
        }
      }
    }
  }
  if (P.conv) {
    // the last CTA to finish re-arms the conversion counter (every warp of every CTA is past its wait by then)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(P.exit_cnt, 1u) + 2u == (unsigned int)P.C) {
        *P.conv_cnt = kSentinel;
        *P.exit_cnt = kSentinel;
      }
    }
  }
  GTSW(2);
#ifdef SBVR_DIAG
  if (P.ts && lane == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    P.ts[((size_t)blockIdx.x * kGW + wib) * 16 + 4] = smid;
    P.ts[((size_t)blockIdx.x * kGW + wib) * 16 + 5] = n;
  }
#endif
}

// ------------------------------------------------------------------ host side
static int group_num_sms() {
  static int nsm[64] = {0};
  const int dev = cur_device();
  if (dev < 0 || dev >= 64) return 148;
  if (!nsm[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    nsm[dev] = v > 0 ? v : 148;
  }
  return nsm[dev];
}

template <int K>
static int occupancy(int smem) {
  cudaFuncSetAttribute(gemv_group_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int o = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, gemv_group_kernel<K>, kGW * 32, smem) != cudaSuccess) {
    cudaGetLastError();
    return kGC;
  }
  return o;
}

struct GroupPlan {
  int n_bands, Us, C;
};
static GroupPlan group_plan(const sbvr_gemv_problem* pr, int n) {
  GroupPlan g{0, 0, 0};
  for (int i = 0; i < n; ++i) {
    g.n_bands += 2 * (pr[i].w.M / 128);
    g.Us += (pr[i].w.M / 128) * (pr[i].w.N / kG);
  }
  // resident CTAs per SM as the hardware reports it (the FP16_Q prologue's arrival count needs the whole grid
  // co-resident; the kernel is persistent anyway)
  static int occ[64] = {0};
  const int dev = cur_device();
  int o = dev >= 0 && dev < 64 ? occ[dev] : 0;
  if (!o) {
    const int smem = pr[0].w.K == 2 ? UnitGeom<2>::kSmem : pr[0].w.K == 3 ? UnitGeom<3>::kSmem : UnitGeom<4>::kSmem;
    if (pr[0].w.K == 2) o = occupancy<2>(smem);
    else if (pr[0].w.K == 3) o = occupancy<3>(smem);
    else o = occupancy<4>(smem);
    if (o < 1) o = 1;
    if (o > kGC) o = kGC;
    if (dev >= 0 && dev < 64) occ[dev] = o;
  }
  int C = group_num_sms() * o;
  const int cap = (g.Us + kPairs - 1) / kPairs;       // at least one unit per warp pair
  g.C = C > cap ? cap : (C < 1 ? 1 : C);
  return g;
}
static size_t group_cnt_bytes(const GroupPlan& g) { return ((size_t)(g.n_bands + 1) * 4 + 255) / 256 * 256; }

template <int K>
static cudaError_t launch_group_k(const GroupParams& P, cudaStream_t st) {
  const int smem = UnitGeom<K>::kSmem;
  static int attr_set[64] = {0};
  const int dev = cur_device();
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemv_group_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.C);
  cfg.blockDim = dim3(kGW * 32);
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

// workspace = [band arrival counters][CTA partial slots: C x 4 x 64 fp32]
//             [SBVR_ACT_FP16_Q scratch: converted planes n_xg x 8 x 4 u32, scales n_xg fp32][conv / exit counters]
// (all 0xFF at rest; every launch leaves it so)
static size_t group_xg(const sbvr_gemv_problem* pr, int n) {
  size_t xg = 0;
  for (int i = 0; i < n; ++i) xg += pr[i].w.N / kG;
  return xg;
}
static size_t group_part_bytes(const grp::GroupPlan& g) { return (size_t)g.C * 4 * 64 * sizeof(float); }
static size_t group_conv_bytes(size_t xg) { return (xg * (8 * 4 * 4 + 4) + 255) / 256 * 256; }

size_t group_workspace_bytes(const sbvr_gemv_problem* pr, int n) {
  const grp::GroupPlan g = grp::group_plan(pr, n);
  return grp::group_cnt_bytes(g) + group_part_bytes(g) + group_conv_bytes(group_xg(pr, n)) + 256;
}

sbvr_status launch_gemv_group(const sbvr_gemv_problem* pr, int n, void* ws, size_t ws_bytes, cudaStream_t st,
                              const GroupPeers* peers) {
  using namespace grp;
  const GroupPlan g = group_plan(pr, n);
  const size_t need = group_workspace_bytes(pr, n);
  if (ws_bytes < need)
    return set_error(SBVR_ERR_WORKSPACE, "gemv_group: workspace %zu bytes < required %zu", ws_bytes, need);
  GroupParams P = {};
  int rbs = 0, uu = 0;
  for (int i = 0; i < n; ++i) {
    P.pr[i].units = pr[i].w.data;
    P.pr[i].xplanes = static_cast<const uint32_t*>(pr[i].x.data);
    P.pr[i].xscales = pr[i].x.scales;
    P.pr[i].Y[0] = pr[i].y;
    P.pr[i].NG = pr[i].w.N / kG;
    P.pr[i].rbbase = rbs;
    P.pr[i].ubase = uu;
    P.ratio_pow[i] = pr[i].w.ratio_pow;
    P.n_ratio[i] = pr[i].w.n_ratio;
    rbs += pr[i].w.M / 128;
    uu += (pr[i].w.M / 128) * (pr[i].w.N / kG);
  }
  P.np = n;
  P.ny = 1;
  if (peers) {                                     // fused all-gather: problem i's y rows -> every rank's full y
    P.ny = peers->n;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < peers->n; ++j) P.pr[i].Y[j] = peers->y[i * peers->n + j] + peers->row_offset[i];
  }
  P.Us = g.Us;
  P.C = g.C;
  P.qq = g.Us / g.C;
  P.rr = g.Us % g.C;
  P.l = pr[0].x.l;
  P.one = 1;
  {
    const char* tsp = getenv("SBVR_TS_PTR");
    P.ts = tsp ? reinterpret_cast<unsigned long long*>(strtoull(tsp, nullptr, 0)) : nullptr;
  }
  char* wsb = reinterpret_cast<char*>(ws);
  P.ws_cnt = reinterpret_cast<unsigned int*>(wsb);
  P.ws_part = reinterpret_cast<float*>(wsb + group_cnt_bytes(g));
  const size_t xg = group_xg(pr, n);
  char* conv = wsb + group_cnt_bytes(g) + group_part_bytes(g);
  P.xq_planes = reinterpret_cast<uint32_t*>(conv);
  P.xq_scales = reinterpret_cast<float*>(conv + xg * 8 * 4 * 4);
  P.conv_cnt = reinterpret_cast<unsigned int*>(conv + group_conv_bytes(xg));
  P.exit_cnt = P.conv_cnt + 1;
  P.conv = pr[0].x.kind == SBVR_ACT_FP16_Q ? 1 : 0;
  P.n_xg = (int)xg;
  {
    int gb = 0;
    for (int i = 0; i < n; ++i) {
      P.gbase[i] = gb;
      if (P.conv) {                                   // the kernel converts x into the workspace and reads it there
        P.xh[i] = static_cast<const uint16_t*>(pr[i].x.data);
        P.pr[i].xplanes = P.xq_planes + (size_t)gb * 4 * P.l;
        P.pr[i].xscales = P.xq_scales + gb;
      }
      gb += pr[i].w.N / kG;
    }
  }
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
