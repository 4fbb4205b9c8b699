// gemv_imma.cu -- SBVR GEMV (§4.4) with the AND+popcount inner products
// executed on the int8 tensor pipe.
//
// The paper's kernel computes, per (row, group), P_tj = popc(beta_t AND d_j) on CUDA cores and
// then sum_t c_t sum_j alpha_j P_tj.  On B200 POPC issues at 16 lanes/clk/SM, which caps that
// formulation near 30% of HBM bandwidth (profiles/r01_step0_microbench.jsonl).  A u8 MMA whose
// operands are single bits IS an AND+popcount: with
//     A[row][k] = bit(beta_t, e(k)) * 2^s        (one LOP3: plane_word & (0x01010101 << s))
//     B[k][j]   = bit(d_j,   e(k)) * 2^(7-s)     (activation plane j, built once per group)
// every product is 128 * (beta AND d), so D[row][j] accumulated over the 128 elements of a
// group is exactly 128 * P_tj.  One mma.m16n8k32.u8 evaluates 16 rows x 8 activation planes x
// 32 elements = 512 weight bits (64 bytes) of AND+popcount; the 8 N-columns of the MMA are the
// l = 8 activation planes, so nothing is wasted at batch 1.
//
// Fragment mapping (mma.m16n8k32, lane = 4*gq + c): a0/a2 = row gq, a1/a3 = row gq+8; a0/a1
// cover k = 4c..4c+3 (bits s of the 4 bytes of word c), a2/a3 k = 16+4c.. (bits s'); four MMAs
// with (s, s') = (0,1), (2,3), (4,5), (6,7) consume all 32 bits of each lane's word, i.e. the
// whole 128-element group of one plane for 16 rows.  The device layout (include/sbvr.h) stores
// each tile in exactly this lane order.
//
// Data movement: each warp streams its own contiguous range of units (band of 4 row tiles x one
// group = 4 KB of planes at K=4 + 320 B of metadata) into a private 3-slot shared-memory ring
// with cp.async.bulk (TMA bulk copies, mbarrier complete_tx); fragments are read with LDS.128.
// This keeps ~8-12 KB in flight per warp without holding prefetch registers.
//
// Epilogue per (row, plane): lane c holds columns j = 2c, 2c+1.  The first MMA of each chain
// adds C = 0x4B400000 (1.5*2^23 as float bits) to column 2c, so u = D0 + kappa*D1 (IMAD, exact,
// kappa = alpha_{2c+1}/alpha_{2c}) reinterpreted as float minus 12582912 is the exact integer
// 128*(P_2c + kappa P_2c+1) without an int->float conversion on the ALU pipe.  Per (row, group):
//     y += s_x * (s * sum_t r^t u_t + b * sum_t u_t)        (c_t = s r^t + b, Eq. 4)
// in packed fp32x2 (rows gq and gq+8 are the two halves).  alpha_{2c}/128 is applied when the
// quad is reduced (2 shuffles per row per 64-row band).
//
// Work split: units are split into contiguous, balanced ranges over 148 x 16 warps.  Bands fully
// inside a warp's range are written directly; a band split across warps is combined
// deterministically by the last-arriving warp (integer counter, partial slots summed in warp
// order).  A band with fewer than 4 row tiles (M % 64 != 0) is handled by a second launch of
// the same kernel instantiated for that band height.
#include <cstdlib>

#include "sbvr_internal.cuh"

namespace sbvr {

constexpr int kImmaWarps = 8;        // warps per CTA
constexpr int kSlots = 2;            // shared-memory ring depth per warp
constexpr int kMaxTT = 4;            // tokens per pass (batched)
constexpr int kBandsPerCta = 4;      // bands a CTA range may touch (host guarantees)
constexpr int kMaxPre = 6;           // later CTAs sharing the owner's last band (host guarantees)

struct ImmaParams {
  const uint8_t* units;     // packed unit records of this launch (full bands, or the tail band)
  const float* ratio_pow;   // [n_ratio][K]
  const uint32_t* xplanes;  // [T][NG][l][4]
  const float* xscales;     // [T][NG]
  float* Y;                 // [T][M]
  int32_t* P;               // debug partials [M][NG][K][l]
  float* ws_part;           // [C][warp][TT][64] partials of each CTA's first band when it is shared
  unsigned int* ws_cnt;     // [C][warp] publish flags (set by the publisher, cleared by the owner)
  int M, N, l, n_ratio;
  int band0;                // first band of this launch
  int Us;                   // units in this launch
  int Pw, qq, rr;           // CTAs and the unit partition over CTAs
  int exp_mode;             // ablation bits (env SBVR_EXP_MODE), 0 in production
  int one;                  // = 1 (runtime value, see i2f_fma)
  unsigned long long* ts;   // phase timestamps (exp_mode & 8)
};
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TS(slot) do { if ((p.exp_mode & 8) && threadIdx.x == 0) p.ts[(size_t)blockIdx.x * 8 + (slot)] = gtime(); } while (0)
#define TSW(slot) do { if ((p.exp_mode & 8) && lane == 0) p.ts[(size_t)blockIdx.x * 8 + (slot)] = gtime(); } while (0)

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
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

// exact int -> float for |u| < 2^22 without the ALU pipe: (u + 0x4B400000) as float - 12582912
__device__ __forceinline__ float i2f_fma(int u, int one) {
  int v;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(v) : "r"(u), "r"(one), "r"(0x4B400000));
  return __int_as_float(v) - 12582912.0f;
}

__device__ __forceinline__ int imad(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int K, int NB>
struct Geom {
  static constexpr int kTileBytes = 256 * K;
  static constexpr int kPlaneBytes = NB * kTileBytes;
  static constexpr int kSbBytes = NB * 64;
  static constexpr int kRiBytes = NB * 16;
  static constexpr int kUnitBytes = kPlaneBytes + kSbBytes + kRiBytes;
  static constexpr int kSlotBytes = (kUnitBytes + 127) / 128 * 128;
  static constexpr int kWarpBytes = kSlots * kSlotBytes;
};

__device__ __forceinline__ int unit_owner(int v, int qq, int rr) {
  const int big = rr * (qq + 1);
  return v < big ? v / (qq + 1) : rr + (v - big) / qq;
}

// one TMA bulk copy per unit: the record [planes][scale/bias][ratio index] is contiguous
template <int K, int NB>
__device__ __forceinline__ void issue_unit(uint8_t* slot, uint64_t* bar, const uint8_t* src) {
  using Gm = Geom<K, NB>;
  constexpr uint32_t bytes = Gm::kPlaneBytes + Gm::kSbBytes + Gm::kRiBytes;
  mbar_expect_tx(bar, bytes);
  bulk_g2s(slot, src, bytes, bar);
}

template <int K, int NB, int TT, bool DEBUG>
__global__ void __launch_bounds__(kImmaWarps * 32, TT == 1 ? 2 : 1) gemv_imma_kernel(ImmaParams p) {
  using Gm = Geom<K, NB>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float s_rat[64];                 // r_i (fp32) for the Horner evaluation of sum_t r^t u_t
  __shared__ uint64_t s_bar[kImmaWarps][kSlots];
  // dynamic smem: [rings][s_part: kBandsPerCta x warps x TT x 64][s_pre: kMaxPre x warps x TT x 64]
  float (*s_part)[kImmaWarps][TT][64] =
      reinterpret_cast<float (*)[kImmaWarps][TT][64]>(smem + kImmaWarps * Gm::kWarpBytes);
  float* s_pre = reinterpret_cast<float*>(smem + kImmaWarps * Gm::kWarpBytes) + kBandsPerCta * kImmaWarps * TT * 64;
  __shared__ int s_pre_ready;
  TS(0);
  // let the next kernel in the stream get scheduled as soon as our CTAs retire
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int i = threadIdx.x; i < p.n_ratio; i += blockDim.x) s_rat[i] = K >= 2 ? p.ratio_pow[i * K + 1] : 0.f;
  for (int i = threadIdx.x; i < kBandsPerCta * kImmaWarps * TT * 64; i += blockDim.x) (&s_part[0][0][0][0])[i] = 0.f;
  if (threadIdx.x == 0) s_pre_ready = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int NG = p.N / kG;
  // CTA range [V0, V1) of units (balanced to +-1 unit), warps take units V0 + wib + 8k
  const int cta = blockIdx.x;
  const int V0 = cta * p.qq + min(cta, p.rr);
  const int V1 = V0 + p.qq + (cta < p.rr ? 1 : 0);
  const int bA = p.band0 + V0 / NG;                 // first band touched by this CTA
  const int bZ = p.band0 + (V1 - 1) / NG;           // last band
  // Bands shared with neighbouring CTAs.  The FIRST contributor owns a shared band (it is the
  // owner's last band, reached at the end of its range); every later contributor has it as its
  // first band, processes it first (natural order) and publishes per-warp partials with release
  // flags as soon as each warp leaves it.  The owner prefetches those partials when it enters
  // the band and adds them in (CTA, warp) order: deterministic, and nobody waits mid-stream.
  const bool pubA = V0 > (bA - p.band0) * NG;                 // bA started in an earlier CTA
  const bool ownZ = V1 < (bZ - p.band0 + 1) * NG && !(bZ == bA && pubA);  // we hold bZ's first unit
  int c_hiZ = cta;                                            // last contributor of an owned bZ
  if (ownZ) c_hiZ = unit_owner((bZ - p.band0 + 1) * NG - 1, p.qq, p.rr);
  const int nPre = ownZ ? (c_hiZ - cta) * kImmaWarps : 0;     // (CTA, warp) partial slots to fetch
  uint8_t* ring = smem + wib * Gm::kWarpBytes;
  uint64_t* bars = s_bar[wib];
  const int n_mine = (V1 - V0 - wib + kImmaWarps - 1) / kImmaWarps;  // units of this warp (may be <= 0)
  // a warp with no unit in the shared first band still publishes (zeros) so the owner's wait ends
  auto publish_zero = [&]() {
    float* slot_p = p.ws_part + ((size_t)cta * kImmaWarps + wib) * (TT * 64);
    for (int e = lane; e < TT * 64; e += 32) slot_p[e] = 0.f;
    __syncwarp();
    if (lane == 0)
      asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(p.ws_cnt + cta * kImmaWarps + wib) : "memory");
  };
  // owner prefetch: acquire the publishers' flags, then copy their slots to shared memory
  auto prefetch_pre = [&]() {
    for (int q = lane; q < nPre; q += 32) {
      unsigned int f = 0;
      long spins = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(p.ws_cnt + cta * kImmaWarps + kImmaWarps + q)
                     : "memory");
        if (++spins > (1L << 28)) __trap();          // a publisher never arrived: fail loudly, never hang
      } while (f == 0u);
    }
    __syncwarp();
    const float* src = p.ws_part + ((size_t)(cta + 1) * kImmaWarps) * (TT * 64);
    for (int e = lane; e < nPre * TT * 64; e += 32) s_pre[e] = __ldcg(src + e);
    if (lane == 0) s_pre_ready = 1;
  };

  if (n_mine > 0) {
    if (lane == 0) {
#pragma unroll
      for (int s2 = 0; s2 < kSlots; ++s2) mbar_init(bars + s2, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
      for (int s2 = 0; s2 < kSlots; ++s2)
        if (s2 < n_mine)
          issue_unit<K, NB>(ring + s2 * Gm::kSlotBytes, bars + s2,
                            p.units + (size_t)(V0 + wib + kImmaWarps * s2) * Gm::kUnitBytes);
    }
    __syncwarp();
    // weights are immutable: their TMA is in flight before we wait for the previous kernel
    // (programmatic dependent launch); activations and the workspace are touched only after.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!DEBUG && pubA && p.band0 + (V0 + wib) / NG != bA) publish_zero();

    // lane constants (Eq. 12: alpha_j = 2^j, alpha_{l-1} = -2^(l-1); MMA columns j0 = 2c, j1 = 2c+1)
    const int j0 = 2 * c, j1 = 2 * c + 1;
    const int al0 = j0 < p.l - 1 ? (1 << j0) : (j0 == p.l - 1 ? -(1 << j0) : 0);
    const int al1 = j1 < p.l - 1 ? (1 << j1) : (j1 == p.l - 1 ? -(1 << j1) : 0);
    const int kappa = al0 != 0 ? al1 / al0 : 0;
    const float lane_scale = (float)al0 * (1.0f / 128.0f);
    const int one = p.one;                          // runtime 1 keeps the conversion IMADs on the FMA pipe
    // lanes whose activation plane gq >= l contribute 0: their B words are masked at use time
    const uint32_t xmask = gq < p.l ? 0xffffffffu : 0u;
    const uint32_t* xlane_ptr = p.xplanes + (gq < p.l ? gq * 4 + c : 0);
    const int xstride = p.l * 4;

    float acc[TT][NB][2];
#pragma unroll
    for (int tk = 0; tk < TT; ++tk)
#pragma unroll
      for (int i = 0; i < NB; ++i) acc[tk][i][0] = acc[tk][i][1] = 0.f;

    int u = V0 + wib;
    int b = p.band0 + u / NG, g = u - (u / NG) * NG;
    int slot = 0;
    uint32_t phase = 0;
    uint32_t Xn[TT];
    float sxn[TT];
#pragma unroll
    for (int tk = 0; tk < TT; ++tk) {
      Xn[tk] = __ldg(xlane_ptr + ((size_t)tk * NG + g) * xstride);
      sxn[tk] = __ldg(p.xscales + (size_t)tk * NG + g);
    }

    for (int k = 0; k < n_mine; ++k) {
      // ---- B operand for group g: activation plane gq, word c, bit-sliced and pre-scaled by 2^(7-s)
      uint32_t Bq[TT][4][2];
      float sx[TT];
#pragma unroll
      for (int tk = 0; tk < TT; ++tk) {
        sx[tk] = sxn[tk];
        const uint32_t X = Xn[tk] & xmask;
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          Bq[tk][pr][0] = bslice(X, 2 * pr);
          Bq[tk][pr][1] = bslice(X, 2 * pr + 1);
        }
      }
      // next unit of this warp (kImmaWarps further): band/group incrementally, activation prefetch
      int gn = g + kImmaWarps, bn = b;
      while (gn >= NG) { gn -= NG; ++bn; }
      const bool has_next = k + 1 < n_mine;
      {
        const int gp = has_next ? gn : g;
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) {
          Xn[tk] = __ldg(xlane_ptr + ((size_t)tk * NG + gp) * xstride);
          sxn[tk] = __ldg(p.xscales + (size_t)tk * NG + gp);
        }
      }

      uint8_t* sl = ring + slot * Gm::kSlotBytes;
      mbar_wait(bars + slot, phase);

#pragma unroll
      for (int i = 0; i < NB; ++i) {
        uint32_t w[2 * K];
        const uint8_t* tb = sl + i * Gm::kTileBytes;
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
          const uint4 v4 = *reinterpret_cast<const uint4*>(tb + q * 512 + lane * 16);
          w[4 * q + 0] = v4.x; w[4 * q + 1] = v4.y; w[4 * q + 2] = v4.z; w[4 * q + 3] = v4.w;
        }
        if (K & 1) {
          const uint2 v2 = *reinterpret_cast<const uint2*>(tb + (K / 2) * 512 + lane * 8);
          w[2 * (K - 1)] = v2.x; w[2 * (K - 1) + 1] = v2.y;
        }
        const uint2 sbp = *reinterpret_cast<const uint2*>(sl + Gm::kPlaneBytes + i * 64 + gq * 8);
        const uint32_t rip = *reinterpret_cast<const uint16_t*>(sl + Gm::kPlaneBytes + Gm::kSbBytes + i * 16 + gq * 2);
        const float r0 = s_rat[rip & 0xffu], r1 = s_rat[rip >> 8];

        // ---- AND + popcount on the tensor pipe: K independent chains (planes) of 4 MMAs
        int D[TT][K][4];
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          const uint32_t m0 = 0x01010101u << (2 * pr), m1 = 0x01010101u << (2 * pr + 1);
#pragma unroll
          for (int t = 0; t < K; ++t) {
            const uint32_t a0 = w[2 * t] & m0, a1 = w[2 * t + 1] & m0, a2 = w[2 * t] & m1, a3 = w[2 * t + 1] & m1;
#pragma unroll
            for (int tk = 0; tk < TT; ++tk) {
              if (pr == 0)
                mma_u8(D[tk][t], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1], 0, 0, 0, 0);
              else
                mma_u8(D[tk][t], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1], D[tk][t][0], D[tk][t][1],
                       D[tk][t][2], D[tk][t][3]);
            }
          }
        }

        if (DEBUG) {
          const int r0w = 64 * b + 16 * i + gq;
#pragma unroll
          for (int t = 0; t < K; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              int32_t* dst = p.P + (((size_t)(r0w + 8 * h) * NG + g) * K + t) * p.l;
              if (j0 < p.l) dst[j0] = D[0][t][2 * h] >> 7;
              if (j1 < p.l) dst[j1] = D[0][t][2 * h + 1] >> 7;
            }
        } else {
          const float s0 = __half2float(__ushort_as_half((unsigned short)(sbp.x & 0xffffu)));
          const float b0 = __half2float(__ushort_as_half((unsigned short)(sbp.x >> 16)));
          const float s1 = __half2float(__ushort_as_half((unsigned short)(sbp.y & 0xffffu)));
          const float b1 = __half2float(__ushort_as_half((unsigned short)(sbp.y >> 16)));
#pragma unroll
          for (int tk = 0; tk < TT; ++tk) {
            // u_t = 128 (P_2c + kappa P_2c+1), exact and |u_t| < 2^22: converted on the FMA pipe as
            // float_bits(u_t + 0x4B400000) - 1.5*2^23 (the ALU pipe is busy with the A extraction)
            float Ph0 = i2f_fma(imad(D[tk][K - 1][1], kappa, D[tk][K - 1][0]), one);
            float Ph1 = i2f_fma(imad(D[tk][K - 1][3], kappa, D[tk][K - 1][2]), one);
            float U0 = Ph0, U1 = Ph1;
#pragma unroll
            for (int t = K - 2; t >= 0; --t) {
              const float f0 = i2f_fma(imad(D[tk][t][1], kappa, D[tk][t][0]), one);
              const float f1 = i2f_fma(imad(D[tk][t][3], kappa, D[tk][t][2]), one);
              Ph0 = fmaf(Ph0, r0, f0);
              Ph1 = fmaf(Ph1, r1, f1);
              U0 += f0;
              U1 += f1;
            }
            acc[tk][i][0] = fmaf(sx[tk], fmaf(s0, Ph0, b0 * U0), acc[tk][i][0]);
            acc[tk][i][1] = fmaf(sx[tk], fmaf(s1, Ph1, b1 * U1), acc[tk][i][1]);
          }
        }
      }

      // ---- release the slot and refill it with this warp's unit k + kSlots
      __syncwarp();
      if (lane == 0 && k + kSlots < n_mine) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_unit<K, NB>(sl, bars + slot, p.units + (size_t)(V0 + wib + kImmaWarps * (k + kSlots)) * Gm::kUnitBytes);
      }
      if (++slot == kSlots) { slot = 0; phase ^= 1u; }

      // ---- leaving band b: reduce the quad; park the 64-row partial in shared memory, or publish it
      if (!DEBUG && (!has_next || bn != b)) {
        const bool publish_now = (b == bA) && pubA;
        float* dst_pub = p.ws_part + ((size_t)cta * kImmaWarps + wib) * (TT * 64);
#pragma unroll
        for (int tk = 0; tk < TT; ++tk)
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            float x0 = acc[tk][i][0] * lane_scale, x1 = acc[tk][i][1] * lane_scale;
            x0 += __shfl_xor_sync(0xffffffffu, x0, 1);
            x1 += __shfl_xor_sync(0xffffffffu, x1, 1);
            x0 += __shfl_xor_sync(0xffffffffu, x0, 2);
            x1 += __shfl_xor_sync(0xffffffffu, x1, 2);
            if (c == 0) {
              float* dst = publish_now ? dst_pub + tk * 64 : &s_part[b - bA][wib][tk][0];
              dst[16 * i + gq] = x0;
              dst[16 * i + gq + 8] = x1;
            }
            acc[tk][i][0] = acc[tk][i][1] = 0.f;
          }
        if (publish_now) {                          // this warp's share of the shared first band
          __syncwarp();
          if (lane == 0)
            asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(p.ws_cnt + cta * kImmaWarps + wib) : "memory");
        }
      }
      // ---- owner of bZ: shortly before the end, fetch the partials the later contributors published
      if (!DEBUG && nPre > 0 && u == max(max(V0, (bZ - p.band0) * NG), V1 - 2 * kImmaWarps)) prefetch_pre();
      b = bn;
      g = gn;
      u += kImmaWarps;
    }
  }
  if (wib == 0) TSW(2);
  if (n_mine <= 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!DEBUG && pubA) publish_zero();
  }
  if (DEBUG) return;
  if (p.exp_mode & 4) return;
  __syncthreads();

  // ---- CTA combine (warp order).  Complete bands and the owned band go to y (the owned band adds
  // the prefetched partials of the later contributors, (CTA, warp) order); a band we published is
  // finished by its owner.
  __syncthreads();
  TS(3);
  if (nPre > 0 && !s_pre_ready && threadIdx.x < 32) prefetch_pre();   // owner had no unit of bZ yet
  __syncthreads();
  const int nbl = bZ - bA + 1;
  for (int e = threadIdx.x; e < nbl * TT * 64; e += blockDim.x) {
    const int bl = e / (TT * 64), tk = (e / 64) % TT, row = e % 64;
    const int bb = bA + bl;
    if (row >= 16 * NB || (bb == bA && pubA)) continue;
    float sum = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < kImmaWarps; ++w2) sum += s_part[bl][w2][tk][row];
    if (bb == bZ && ownZ)
      for (int q = 0; q < nPre; ++q) sum += s_pre[(q * TT + tk) * 64 + row];
    p.Y[(size_t)tk * p.M + 64 * bb + row] = sum;
  }
  if (nPre > 0) {                                   // reset the consumed flags for the next launch
    for (int q = threadIdx.x; q < nPre; q += blockDim.x) p.ws_cnt[cta * kImmaWarps + kImmaWarps + q] = 0u;
  }
  TS(4);
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct Plan {
  int NG, MT, n_full, tail_nb, n_bands;
  int Us_main, C_main, Us_tail, C_tail;
};

// CTAs per launch: 2 per SM (one wave at 16 warps/SM), but at least enough that a CTA range
// of units touches at most kBandsPerCta bands, and never more CTAs than units.
static int ctas_for(int Us, int NG) {
  if (Us <= 0) return 0;
  int C = 2 * num_sms();
  const int max_range = (kBandsPerCta - 1) * NG;  // a range of <= max_range units touches <= kBandsPerCta bands
  const int need = (Us + max_range - 1) / max_range + 1;
  if (C < need) C = need;
  // a band may be shared by at most kMaxPre + 1 CTAs: ranges of >= ceil(NG / kMaxPre) units
  const int min_range = (NG + kMaxPre - 1) / kMaxPre;
  const int cap = Us / min_range;
  if (C > cap && cap >= 1) C = cap;
  if (C > Us) C = Us;
  if (C < 1) C = 1;
  return C;
}

static Plan make_plan(const sbvr_weights* w) {
  Plan pl;
  pl.NG = w->N / kG;
  pl.MT = w->M / kTileRows;
  pl.n_full = pl.MT / 4;
  pl.tail_nb = pl.MT % 4;
  pl.n_bands = pl.n_full + (pl.tail_nb ? 1 : 0);
  pl.Us_main = pl.n_full * pl.NG;
  pl.C_main = ctas_for(pl.Us_main, pl.NG);
  pl.Us_tail = pl.tail_nb ? pl.NG : 0;
  pl.C_tail = ctas_for(pl.Us_tail, pl.NG);
  return pl;
}

// workspace = [flags: one u32 per (CTA, warp)][published partials: TT x 64 floats per (CTA, warp)]
size_t imma_workspace_bytes(const sbvr_weights* w, int T) {
  const Plan pl = make_plan(w);
  const int TT = T < kMaxTT ? T : kMaxTT;
  const int C = pl.C_main > pl.C_tail ? pl.C_main : pl.C_tail;
  const size_t flags = ((size_t)C * kImmaWarps * 4 + 255) / 256 * 256;
  return flags + (size_t)C * kImmaWarps * TT * 64 * sizeof(float);
}

template <int K, int NB, int TT, bool DEBUG>
static cudaError_t launch_one(const ImmaParams& p, cudaStream_t st) {
  const int smem = kImmaWarps * Geom<K, NB>::kWarpBytes + (kBandsPerCta + kMaxPre) * kImmaWarps * TT * 64 * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemv_imma_kernel<K, NB, TT, DEBUG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.Pw);
  cfg.blockDim = dim3(kImmaWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemv_imma_kernel<K, NB, TT, DEBUG>, p);
}

template <int K, int NB>
static cudaError_t launch_nb(const ImmaParams& p, int TT, bool debug, cudaStream_t st) {
  if (debug) return launch_one<K, NB, 1, true>(p, st);
  switch (TT) {
    case 1: return launch_one<K, NB, 1, false>(p, st);
    case 2: return launch_one<K, NB, 2, false>(p, st);
    default: return launch_one<K, NB, 4, false>(p, st);
  }
}

template <int K>
static cudaError_t launch_k(const ImmaParams& p, int NB, int TT, bool debug, cudaStream_t st) {
  switch (NB) {
    case 4: return launch_nb<K, 4>(p, TT, debug, st);
    case 3: return launch_nb<K, 3>(p, TT, debug, st);
    case 2: return launch_nb<K, 2>(p, TT, debug, st);
    default: return launch_nb<K, 1>(p, TT, debug, st);
  }
}

static cudaError_t launch_any(int K, const ImmaParams& p, int NB, int TT, bool debug, cudaStream_t st) {
  switch (K) {
    case 1: return launch_k<1>(p, NB, TT, debug, st);
    case 2: return launch_k<2>(p, NB, TT, debug, st);
    case 3: return launch_k<3>(p, NB, TT, debug, st);
    case 4: return launch_k<4>(p, NB, TT, debug, st);
    case 5: return launch_k<5>(p, NB, TT, debug, st);
    case 6: return launch_k<6>(p, NB, TT, debug, st);
    case 7: return launch_k<7>(p, NB, TT, debug, st);
    default: return launch_k<8>(p, NB, TT, debug, st);
  }
}

sbvr_status launch_gemv_imma(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                             int32_t* P_debug, cudaStream_t st) {
  const Plan pl = make_plan(w);
  ImmaParams p;
  const Layout Lo(w->M, w->N, w->K);
  p.ratio_pow = w->ratio_pow;
  p.M = w->M; p.N = w->N; p.l = x->l; p.n_ratio = w->n_ratio;
  p.P = P_debug;
  p.one = 1;
  {
    const char* em = getenv("SBVR_EXP_MODE");
    p.exp_mode = em ? atoi(em) : 0;
    const char* tsp = getenv("SBVR_TS_PTR");
    p.ts = tsp ? reinterpret_cast<unsigned long long*>(strtoull(tsp, nullptr, 0)) : nullptr;
    if (!p.ts) p.exp_mode &= ~8;
  }
  const int Cmax = pl.C_main > pl.C_tail ? pl.C_main : pl.C_tail;
  const size_t cnt_bytes = ((size_t)Cmax * kImmaWarps * 4 + 255) / 256 * 256;
  p.ws_cnt = ws ? reinterpret_cast<unsigned int*>(ws) : nullptr;
  p.ws_part = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + cnt_bytes) : nullptr;
  (void)ws_bytes;
  const uint32_t* xp = static_cast<const uint32_t*>(x->data);
  const bool debug = P_debug != nullptr;
  int done = 0;
  while (done < T) {
    const int rem = T - done;
    const int TT = debug ? 1 : (rem >= 4 ? 4 : (rem >= 2 ? 2 : 1));
    p.xplanes = xp + (size_t)done * pl.NG * x->l * 4;
    p.xscales = x->scales + (size_t)done * pl.NG;
    p.Y = Y ? Y + (size_t)done * w->M : nullptr;
    for (int part = 0; part < 2; ++part) {
      const int NB = part == 0 ? 4 : pl.tail_nb;
      const int Us = part == 0 ? pl.Us_main : pl.Us_tail;
      if (Us == 0) continue;
      p.band0 = part == 0 ? 0 : pl.n_full;
      p.units = w->data + (part == 0 ? 0 : Lo.unit_off(pl.n_full, 0));
      p.Us = Us;
      p.Pw = part == 0 ? pl.C_main : pl.C_tail;
      p.qq = Us / p.Pw;
      p.rr = Us % p.Pw;
      cudaError_t e = launch_any(w->K, p, NB, TT, debug, st);
      if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "gemv_imma setup: %s", cudaGetErrorString(e));
      sbvr_status s = check_launch("gemv_imma_kernel");
      if (s != SBVR_OK) return s;
    }
    if (debug) break;
    done += TT;
  }
  return SBVR_OK;
}

}  // namespace sbvr
