// gemv_mma.cuh -- the batch-1..8 mma.sync SBVR GEMV kernel template (see the description below) and its
// launchers; instantiated per K in gemv_mma_k<K>.cu (parallel compilation), dispatched by gemv_mma.cu.
// gemv_mma.cu -- SBVR GEMV at batch 1-3 (§4.4): the AND+popcount inner
// products on the int8 tensor pipe through warp-level mma.sync (IMMA.16832), the path with the
// highest instruction throughput when the activation side is only l = 8 bit-planes wide.
//
// The paper's kernel computes, per (row, group), P_tj = popc(beta_t AND d_j) on CUDA cores and
// then sum_t c_t sum_j alpha_j P_tj.  On B200 POPC issues at 16 lanes/clk/SM, which caps that
// formulation near 30% of HBM bandwidth (profiles/r01_step0_microbench.jsonl); tcgen05.mma
// kind::i8 costs a flat ~46 cycles per M=128 instruction for any N <= 64
// (profiles/r01_tc_rate.jsonl), too slow when N = 8.  A u8 MMA whose operands are single bits IS
// an AND+popcount: with
//     A[row][k] = bit(beta_t, e(k)) * 2^s        (one LOP3: plane_word & (0x01010101 << s))
//     B[k][j]   = bit(d_j,   e(k)) * 2^(7-s)     (activation plane j, built once per group)
// every product is 128 * (beta AND d), so D[row][j] accumulated over the 128 elements of a
// group is exactly 128 * P_tj.  One mma.m16n8k32.u8 evaluates 16 rows x 8 activation planes x
// 32 elements = 512 weight bits (64 bytes) of AND+popcount.
//
// Fragment mapping (mma.m16n8k32, lane = 4*gq + c): a0/a2 = row gq, a1/a3 = row gq+8; a0/a1
// cover k = 4c..4c+3 (bits s of the 4 bytes of word c), a2/a3 k = 16+4c.. (bits s'); four MMAs
// with (s, s') = (0,1), (2,3), (4,5), (6,7) consume all 32 bits of each lane's word, i.e. the
// whole 128-element group of one plane for 16 rows.  Lane (gq, c) gathers word c of its two
// rows with LDS.32 from the row-major unit record (sbvr.h); the chunk swizzle makes the 32 lanes
// hit 32 distinct banks.
//
// Data movement: a "band" is one 64-row half of a 128-row block; each warp streams its own
// contiguous range of (band, group) units (4 KB of planes at K=4 + 320 B of metadata, three
// cp.async.bulk copies) into a private 2-slot shared-memory ring (mbarrier complete_tx).
//
// Epilogue per (row, plane): lane c holds columns j = 2c, 2c+1, u = D0 + kappa*D1 (IMAD, exact,
// kappa = alpha_{2c+1}/alpha_{2c}), converted exactly on the FMA pipe with the 1.5*2^23 magic
// number, y += s_x * (s * sum_t r^t u_t + b * sum_t u_t) (c_t = s r^t + b, Eq. 4);
// alpha_{2c}/128 is applied when the quad is reduced (2 shuffles per row per band).
//
// Work split: units are split into contiguous, balanced ranges over CTAs (two 8-warp CTAs per SM: when
// one finishes, a CTA of the next launch starts its weight copies on that half SM while the other still runs),
// and each CTA's tiles into contiguous warp ranges.  A band shared by several warps is summed in
// warp order by the last warp to finish it (smem counter); a band shared by several CTAs by the
// last CTA to finish it (global arrival counter; every contributor publishes its partial first):
// the sum runs in CTA order whoever arrives last, so y is deterministic, and no CTA ever waits for
// another (no co-residency assumption).  A band with fewer than 4 row tiles (M % 64 != 0) is
// handled by a second launch instantiated for that band height.


#pragma once
#include <cstdlib>
#include <type_traits>

#include "sbvr_internal.cuh"

namespace sbvr {
namespace mma {

inline int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}


#ifndef SBVR_MMA_WARPS
#define SBVR_MMA_WARPS 8
#endif
constexpr int kImmaWarps = SBVR_MMA_WARPS;   // warps per CTA (two CTAs per SM fill the register file)
#ifndef SBVR_MMA_MIN_UNITS
#define SBVR_MMA_MIN_UNITS 4
#endif
constexpr int kMinUnitsPerCta = SBVR_MMA_MIN_UNITS;   // small problems: spread over SMs, at least this many units per CTA
#ifndef SBVR_MMA_CTAS_PER_SM
#define SBVR_MMA_CTAS_PER_SM 2     // resident CTAs per SM: two 8-warp CTAs (profiles/r02_cta_shape_ab.txt)
#endif
#ifndef SBVR_MMA_OWNER_PULL
#define SBVR_MMA_OWNER_PULL 0
#endif
#ifndef SBVR_MMA_SLOTS
#define SBVR_MMA_SLOTS 2
#endif
constexpr int kSlots = SBVR_MMA_SLOTS;   // shared-memory ring depth per warp
// weight copies a warp issues at launch; the rest of the ring is filled when the first unit lands (a smaller
// initial burst lets the first units arrive sooner, so compute overlaps the stream)
#ifndef SBVR_MMA_INIT_SLOTS
#define SBVR_MMA_INIT_SLOTS SBVR_MMA_SLOTS
#endif
constexpr int kInitSlots = SBVR_MMA_INIT_SLOTS;
constexpr int kMaxTT = 4;            // tokens per pass (batched)
constexpr int kZbMinT = 3;           // SBVR-x batches from this T use the z-column formulation (8 tokens per pass)
constexpr int kSumBatchMax = 8;      // CTA partials loaded per batch by a band's owner (x TT words per lane)
constexpr unsigned int kSentinel = 0xFFFFFFFFu;   // "not yet written" (a NaN arithmetic never produces)

struct ImmaParams {
  const uint8_t* units;     // the weights' unit records (sbvr.h)
  const float* ratio_pow;   // [n_ratio][K]
  const uint32_t* coef_table;   // SBVR_META_INDEXED: [1 + 2 n] (n, then (s16 | b16 << 16, ratio index)); else NULL
  const uint16_t* xq;       // XQ: fp16 x [N] converted to SBVR-x (Eq. 12) in the prologue; else NULL
  int xq_groups;            // XQ: groups converted per CTA (shared-memory rows)
  const uint32_t* xplanes;  // [T][NG][l][4] (SBVR-x)
  const uint16_t* xh;       // [T][N] fp16 x (fp16-x path)
  int ntok;                 // fp16-x: tokens in this pass (<= 8, one per MMA column)
  const float* xscales;     // [T][NG]
  float* Y;                 // [T][M] (when n_peers == 0)
  float* peer_y[8];         // fused row-shard all-gather: y goes to every rank's full-y buffer [T][M_full] at row
  int n_peers, y_off, M_full;   // offset y_off (symmetric-memory peer pointers; dist.py)
  int32_t* P;               // debug partials [M][NG][K][l]
  float* ws_part;           // [CTA][2][TT][64] partials of a CTA's first / last band when other CTAs share it
                            // (kSentinel words at rest: sbvr_workspace_init, re-armed by the band's reducer)
  unsigned int* ws_cnt;     // [global band] arrival counters, 0xFFFFFFFF at rest (reset by the band's reducer)
  int M, N, l, n_ratio;
  int band0;                // first band of this launch
  int K, n_full, tail_rows; // row blocks: full ones, rows of the tail block
  int Us;                   // units in this launch
  int Pw, qq, rr;           // CTAs and the unit partition over CTAs
  int one;                  // = 1 (runtime value, see i2f_fma)
  // chain hint (sbvr_gemv_chain): the next GEMV's weights and its work partition (main launch), or NULL
  const uint8_t* nx_units;
  int nx_NG, nx_K, nx_Us, nx_C, nx_qq, nx_rr;
  int fine;                 // 1: warp ranges at single-tile granularity (large problems: the last step of a
                            // warp may be a lone tile); 0: whole tile pairs (small problems keep the ILP)
  int exp;                  // ablation bits (env SBVR_EXP_MODE, 0 in production): 1 skip the tile
                            // compute, 2 compute only (no TMA: stale shared memory), 4 skip the
                            // band flush, 8 exit right after the prologue
  unsigned long long* ts;   // diagnostics (env SBVR_TS_PTR): [CTA][warp][8] stamps 0-3, smid, units
};
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Diagnostics (ablation switches, per-warp timestamps) exist only in a -DSBVR_DIAG build (tools/build_var.sh):
// the production kernel carries no runtime checks for them.
#ifdef SBVR_DIAG
#define TSW(slot) do { if (p.ts && lane == 0) p.ts[((size_t)blockIdx.x * kImmaWarps + wib) * 8 + (slot)] = gtime(); } while (0)
#define EXPM(bit) (p.exp & (bit))
#else
#define TSW(slot) do { } while (0)
#define EXPM(bit) 0
#endif

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

__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1, int c0, int c1, int c2, int c3) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}
// w >> s for a compile-time s after unrolling, on the FMA pipe (IMAD.HI) instead of the ALU
__device__ __forceinline__ uint32_t shr_u(uint32_t w, int s) { return s == 0 ? w : __umulhi(w, 1u << (32 - s)); }

__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// fp16-x A operand: bits s and 16+s of plane word w as the fp16 pair (bit_s ? 1.0 : 0, bit_16+s ? 1.0 : 0):
// mask (one LOP3), then one IMAD by 0x3C00 >> s turns each isolated bit into 0x3C00 (no carry between
// halves).  Bits 11..15 are taken from w >> 5 so the multiplier stays an integer.
__device__ __forceinline__ uint32_t f16_bits(uint32_t w, uint32_t w5, int S) {   // S is a constant after unrolling
  if (S <= 10) return (w & (0x00010001u << S)) * (0x3C00u >> S);
  return (w5 & (0x00010001u << (S - 5))) * (0x3C00u >> (S - 5));
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

template <int K, int NB, bool IDX = false>
struct Geom {
  static constexpr int kTileBytes = 256 * K;
  static constexpr int kPlaneBytes = NB * kTileBytes;
  static constexpr int kSbBytes = IDX ? 0 : NB * 64;   // IDX (SBVR_META_INDEXED): no per-group s/b, a table index
  static constexpr int kRiBytes = NB * 16;
  static constexpr int kUnitBytes = kPlaneBytes + kSbBytes + kRiBytes;
  static constexpr int kSlotBytes = (kUnitBytes + 127) / 128 * 128;
  static constexpr int kWarpBytes = kSlots * kSlotBytes;
};

__device__ __forceinline__ uint32_t ld_relaxed(const float* ptr) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

// y store: local Y, or (fused all-gather epilogue) the same value into every rank's full y over NVLink
__device__ __forceinline__ void store_y(const ImmaParams& p, int tk, int row, float v) {
  if (p.n_peers == 0) {
    p.Y[(size_t)tk * p.M + row] = v;
  } else {
#pragma unroll 1
    for (int j = 0; j < p.n_peers; ++j) p.peer_y[j][(size_t)tk * p.M_full + p.y_off + row] = v;
  }
}

__device__ __forceinline__ int unit_owner(int v, int qq, int rr) {
  const int big = rr * (qq + 1);
  return v < big ? v / (qq + 1) : rr + (v - big) / qq;
}

// a band is the half h of row block rb: its planes, scale/bias and ratio indices are three
// contiguous pieces of the (rb, g) unit record.  Tiles [i0, i1) of the band -> three bulk copies
// into the slot at their full-unit offsets [planes][sb][ri].
template <int K, int NB, bool IDX = false>
__device__ __forceinline__ void issue_unit(uint8_t* slot, uint64_t* bar, const ImmaParams& p, int band, int g,
                                           int i0, int i1) {
  using Gm = Geom<K, NB, IDX>;
  constexpr int kMeta = IDX ? 1 : 5;           // meta bytes per row: table index, or fp16 s, b + ratio index
  const int NG = p.N / kG;
  const int rb = band >> 1, h = band & 1;
  const int R = rb < p.n_full ? 128 : p.tail_rows;
  const size_t ub = (size_t)R * (16 * K + kMeta);
  const uint8_t* u = rb < p.n_full ? p.units + ((size_t)rb * NG + g) * ub
                                    : p.units + (size_t)p.n_full * NG * (128 * (16 * K + kMeta)) + (size_t)g * ub;
  const int r0 = 64 * h + 16 * i0, nt = i1 - i0;
  mbar_expect_tx(bar, nt * (Gm::kTileBytes + (IDX ? 16 : 64 + 16)));
  bulk_g2s(slot + i0 * Gm::kTileBytes, u + (size_t)r0 * 16 * K, nt * Gm::kTileBytes, bar);
  if (!IDX) bulk_g2s(slot + Gm::kPlaneBytes + 64 * i0, u + (size_t)R * 16 * K + 4 * r0, nt * 64, bar);
  bulk_g2s(slot + Gm::kPlaneBytes + Gm::kSbBytes + 16 * i0, u + (size_t)R * (16 * K + kMeta - 1) + r0, nt * 16, bar);
}

// Eq. 12 for the activation groups gi = first, first + stride, ... < n of this CTA (group g0 + gi mod NG) by one
// warp, bit-identical to encode_vector_kernel (the same fp32 IEEE ops): absmax -> s_x = absmax / (2^(l-1) - 1)
// (__fdiv_rn), z = clamp(rne(x / s_x)), l-bit two's-complement planes by ballot; word (plane j, 32-element word c)
// -> out[32 gi + 4 j + c], s_x -> out_s[gi].  The loads of up to four groups are issued before any arithmetic,
// so a warp pays the L2 latency once per four groups.
__device__ __forceinline__ void xq_convert_groups(const ImmaParams& p, int g0, int NG, int first, int stride, int n,
                                                  uint32_t* out, float* out_s) {
  const int lane = threadIdx.x & 31;
  const int zmax = (1 << (p.l - 1)) - 1;
  const uint32_t lmask = (1u << p.l) - 1u;
  for (int gb = first; gb < n; gb += 4 * stride) {
    float v[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gi = gb + q * stride;
      int g = g0 + gi;
      if (g >= NG) g -= NG;
      const uint16_t* xg = p.xq + (size_t)g * kG;
#pragma unroll
      for (int c = 0; c < 4; ++c) v[q][c] = gi < n ? __half2float(__ushort_as_half(__ldg(xg + 32 * c + lane))) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gi = gb + q * stride;
      if (gi >= n) break;
      float a = fmaxf(fmaxf(fabsf(v[q][0]), fabsf(v[q][1])), fmaxf(fabsf(v[q][2]), fabsf(v[q][3])));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
      const float sx = (a != 0.0f) ? __fdiv_rn(a, (float)zmax) : 0.0f;
      uint32_t mine = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        int z = 0;
        if (sx != 0.0f) {
          z = __float2int_rn(__fdiv_rn(v[q][c], sx));
          z = min(max(z, -zmax), zmax);
        }
        const uint32_t u = (uint32_t)z & lmask;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t word = __ballot_sync(0xffffffffu, (u >> j) & 1u);
          if (lane == 4 * j + c) mine = word;
        }
      }
      out[32 * gi + lane] = lane < 4 * p.l ? mine : 0u;
      if (lane == 0) out_s[gi] = sx;
    }
  }
}

// L2 prefetch of the first two units warp wib of CTA c will copy in the next GEMV of a chain (same unit-record
// layout and work split as this kernel's main launch, SBVR_META_GROUP): cp.async.bulk.prefetch.L2, no smem.
// (scalar arguments only: taking the address of the kernel's parameter struct would move it to local memory)
static __device__ __noinline__ void prefetch_next(const uint8_t* nx_units, int nx_NG, int K, int nx_C, int nx_qq,
                                                  int nx_rr, int c, int wib) {
  if (c >= nx_C) return;
  const int V0 = c * nx_qq + min(c, nx_rr);
  const int V1 = V0 + nx_qq + (c < nx_rr ? 1 : 0);
  const int nTc = (V1 - V0) * 4;
  const int tq = nTc / kImmaWarps, tr = nTc % kImmaWarps;
  const int T0 = wib * tq + min(wib, tr), T1 = T0 + tq + (wib < tr ? 1 : 0);
  if (T1 <= T0) return;
  const size_t ub = (size_t)128 * (16 * K + 5);
  for (int uu = V0 + T0 / 4; uu <= V0 + (T1 - 1) / 4 && uu < V0 + T0 / 4 + 2; ++uu) {
    const int band = uu / nx_NG, g = uu - band * nx_NG;
    const int rb = band >> 1, h = band & 1;
    const uint8_t* u = nx_units + ((size_t)rb * nx_NG + g) * ub;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)h * 64 * 16 * K), "r"(64 * 16 * K)
                 : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)128 * 16 * K + h * 256), "r"(256)
                 : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)128 * (16 * K + 4) + h * 64), "r"(64)
                 : "memory");
  }
}

// F16X: the fp16-x path (north star): M_t = sum_e beta_t[e] x_e with x in fp16, on
// mma.m16n8k16 f16 (A = plane bits as 0/1.0 pairs, B = the lane's own x values, columns = tokens);
// TT is then the number of token columns kept (<= 8).
template <int K, int NB, int TT, bool DEBUG, bool F16X, bool ZB, bool IDX, bool XQ>
#ifdef SBVR_MMA_MAXNREG
__global__ void __maxnreg__(SBVR_MMA_MAXNREG) gemv_mma_kernel(ImmaParams p) {
#else
__global__ void __launch_bounds__(kImmaWarps * 32, SBVR_MMA_CTAS_PER_SM) gemv_mma_kernel(ImmaParams p) {
#endif
  using Gm = Geom<K, NB, IDX>;
  constexpr int PTC = (NB % 2 == 0 && ((TT == 1 && !F16X) || ZB)) ? 2 : 1;   // tiles per compute step
  constexpr int NACC = (F16X || ZB) ? 2 : TT;          // accumulators per tile: tokens (SBVR) or columns (F16X, ZB)
  constexpr int NMMA = ZB ? 1 : TT;                    // MMAs per (tile, plane, slice pair)
  constexpr int kSumBatch = kSumBatchMax / (TT >= 4 ? 4 : TT);   // keep the pulled words <= 16 per lane
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float s_rat[64];                 // r_i (fp32) for the Horner evaluation of sum_t r^t u_t
  __shared__ __align__(8) uint32_t s_tab[IDX ? 2 * 256 : 2];   // IDX: coefficient table (fp16 s | b << 16, r fp32)
  __shared__ uint64_t s_bar[kImmaWarps][kSlots];
  __shared__ unsigned int s_cnt[2 * kImmaWarps];  // warps done with a band, by (first warp, its first/last band)
  __shared__ int s_fb[kImmaWarps];                 // first launch-local band of each warp
  __shared__ int s_lb[kImmaWarps];                 // last launch-local band of each warp (-1: no tiles)
  // dynamic smem: [rings][s_part: warps x 2 (first / last band) x TT x 64]
  float* s_part = reinterpret_cast<float*>(smem + kImmaWarps * Gm::kWarpBytes);
  // XQ: this CTA's activation groups converted in the prologue (Eq. 12): [groups][8 planes][4 words] + scales
  uint32_t* s_xq = reinterpret_cast<uint32_t*>(s_part + kImmaWarps * 2 * TT * 64);
  float* s_xqs = reinterpret_cast<float*>(s_xq + 32 * p.xq_groups);
  // let the next kernel in the stream get scheduled as soon as our CTAs retire
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int NG = p.N / kG;
  TSW(0);
  // CTA range [V0, V1) of units (balanced to +-1 unit); its NB-tile units are split over the
  // warps at tile granularity: warp w takes the contiguous CTA-local tiles [T0, T1)
  const int cta = blockIdx.x;
  const int V0 = cta * p.qq + min(cta, p.rr);
  const int V1 = V0 + p.qq + (cta < p.rr ? 1 : 0);
  const int bA = V0 / NG;                              // first launch-local band of this CTA
  // (warp ranges at tile granularity; the compute loop takes PTC = 2 tiles per step where it can)
  const int gran = p.fine ? 1 : PTC;                  // split granularity (tiles)
  const int nTc = (V1 - V0) * NB / gran;
  const int tq = nTc / kImmaWarps, tr = nTc % kImmaWarps;
  const int T0 = gran * (wib * tq + min(wib, tr)), T1 = T0 + gran * (tq + (wib < tr ? 1 : 0));
  const int n_mine = T1 > T0 ? (T1 - 1) / NB - T0 / NB + 1 : 0;   // units this warp touches
  const int uf = V0 + T0 / NB;                          // its first unit
  auto tiles_of = [&](int k, int& i0, int& i1) {        // tiles of the warp's k-th unit
    i0 = k == 0 ? T0 % NB : 0;
    i1 = k == n_mine - 1 ? (T1 - 1) % NB + 1 : NB;
  };
  uint8_t* ring = smem + wib * Gm::kWarpBytes;
  uint64_t* bars = s_bar[wib];
  int ib_band = uf / NG, ib_g = uf - (uf / NG) * NG;   // lane 0: (band, group) of the next unit to fetch
  auto issue_next = [&](uint8_t* slot_ptr, uint64_t* bar, int kk) {
    int i0, i1;
    tiles_of(kk, i0, i1);
    issue_unit<K, NB, IDX>(slot_ptr, bar, p, p.band0 + ib_band, ib_g, i0, i1);
    if (++ib_g == NG) { ib_g = 0; ++ib_band; }
  };
  if (n_mine > 0 && lane == 0) {
    // weights are immutable: their TMA starts before we wait for the previous kernel
#pragma unroll
    for (int s2 = 0; s2 < kSlots; ++s2) mbar_init(bars + s2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s2 = 0; s2 < kSlots; ++s2)
      if (s2 < kInitSlots && s2 < n_mine && !EXPM(2)) issue_next(ring + s2 * Gm::kSlotBytes, bars + s2, s2);
  }
  for (int i = threadIdx.x; i < p.n_ratio; i += blockDim.x) s_rat[i] = K >= 2 ? p.ratio_pow[i * K + 1] : 0.f;
  if constexpr (IDX)      // entry e -> (fp16 s | b << 16, r as fp32 bits): one 8-byte shared load per row and tile
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
      const bool live = i < (int)p.coef_table[0];
      s_tab[2 * i] = live ? p.coef_table[1 + 2 * i] : 0u;
      s_tab[2 * i + 1] = live ? __float_as_uint(K >= 2 ? p.ratio_pow[p.coef_table[2 + 2 * i] * K + 1] : 0.f) : 0u;
    }
  for (int i = threadIdx.x; i < 2 * kImmaWarps; i += blockDim.x) s_cnt[i] = 0u;
  if (threadIdx.x < kImmaWarps) {
    const int w2 = threadIdx.x;
    const int t0 = gran * (w2 * tq + min(w2, tr)), t1 = t0 + gran * (tq + (w2 < tr ? 1 : 0));
    s_fb[w2] = t1 > t0 ? (V0 + t0 / NB) / NG : 0x7fffffff;
    s_lb[w2] = t1 > t0 ? (V0 + (t1 - 1) / NB) / NG : -1;
  }
  __syncthreads();
  // XQ: groups g0, g0+1, ... (mod NG) of this CTA's unit range, converted by its warps (one warp per group)
  const int xq_g0 = V0 % NG;
  const int xq_n = min(V1 - V0, NG);
  if constexpr (XQ) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // x is produced by the previous kernel
    xq_convert_groups(p, xq_g0, NG, wib, kImmaWarps, xq_n, s_xq, s_xqs);
    __syncthreads();
  }
  if (n_mine <= 0) return;
  if constexpr (!XQ) asm volatile("griddepcontrol.wait;" ::: "memory");   // activations / workspace / y from here
  if (EXPM(8)) return;

  // lane constants (Eq. 12: alpha_j = 2^j, alpha_{l-1} = -2^(l-1); MMA columns j0 = 2c, j1 = 2c+1)
  const int j0 = 2 * c, j1 = 2 * c + 1;
  const int al0 = j0 < p.l - 1 ? (1 << j0) : (j0 == p.l - 1 ? -(1 << j0) : 0);
  const int al1 = j1 < p.l - 1 ? (1 << j1) : (j1 == p.l - 1 ? -(1 << j1) : 0);
  const int kappa = al0 != 0 ? al1 / al0 : 0;
  const float lane_scale = (float)al0 * (1.0f / 128.0f);
  // u = D0 + kappa*D1 (exact int, |u| < 2^22) is converted on the FMA pipe: (u + 0x4B400000) read as
  // a float is 1.5*2^23 + u exactly, minus 1.5*2^23 (FADD2 for the two rows of the lane)
  const int magic = 0x4B400000;
  const float2 cmagic = make_float2(12582912.0f, 12582912.0f);
  // lanes whose activation plane gq >= l contribute 0: their B words are masked at use time
  const uint32_t xmask = gq < p.l ? 0xffffffffu : 0u;
  const uint32_t* xlane_ptr = p.xplanes + (gq < p.l ? gq * 4 + c : 0);
  const int xstride = p.l * 4;
  // chunk swizzle of rows gq and gq+8 (sbvr.h; depends on the low 3 row bits only)
  const int swz_a = chunk_swizzle(K, gq), swz_b = chunk_swizzle(K, gq + 8);

  float2 acc[NACC][NB];
#pragma unroll
  for (int tk = 0; tk < NACC; ++tk)
#pragma unroll
    for (int i = 0; i < NB; ++i) acc[tk][i] = make_float2(0.f, 0.f);

  int u = uf;
  int b = u / NG, g = u - b * NG;
  int slot = 0;
  uint32_t phase = 0;
  uint32_t Xn[TT];
  float sxn[TT];
  uint4 Xh[F16X ? 4 : 1];                              // fp16-x: x[token gq][32c .. 32c+31] of the group
  uint32_t Xz[ZB ? 8 : 1];                             // ZB: word c of the 8 planes of token gq (sign-extended)
  float sxz[2];                                        // ZB: scales of this lane's output tokens 2c, 2c+1
  auto load_xz = [&](int gg) {
    if constexpr (ZB) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        Xz[j] = gq < p.ntok ? __ldg(p.xplanes + (((size_t)gq * NG + gg) * p.l + min(j, p.l - 1)) * 4 + c) : 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) sxz[h] = 2 * c + h < p.ntok ? __ldg(p.xscales + (size_t)(2 * c + h) * NG + gg) : 0.f;
    }
  };
  auto load_xh = [&](int gg) {
    if constexpr (F16X) {
      if (gq < p.ntok) {
        const uint4* src = reinterpret_cast<const uint4*>(p.xh + (size_t)gq * p.N + (size_t)gg * kG + 32 * c);
#pragma unroll
        for (int q = 0; q < 4; ++q) Xh[q] = __ldg(src + q);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) Xh[q] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  };
  if constexpr (F16X) {
    load_xh(g);
  } else if constexpr (ZB) {
    load_xz(g);
  } else if constexpr (XQ) {
    const int gi = g >= xq_g0 ? g - xq_g0 : g - xq_g0 + NG;
    Xn[0] = gq < p.l ? s_xq[32 * gi + 4 * gq + c] : 0u;
    sxn[0] = s_xqs[gi];
  } else {
#pragma unroll
    for (int tk = 0; tk < TT; ++tk) {
      Xn[tk] = __ldg(xlane_ptr + ((size_t)tk * NG + g) * xstride);
      sxn[tk] = __ldg(p.xscales + (size_t)tk * NG + g);
    }
  }

  for (int k = 0; k < n_mine; ++k) {
    // ---- B operand for group g: activation plane gq, word c, bit-sliced and pre-scaled by 2^(7-s)
    uint32_t Bq[NMMA][4][2];
    float sx[TT];
    float sxc[2];
    uint32_t Bh[F16X ? 8 : 1][2];                       // fp16-x B: (x_s, x_16+s) pairs for s = 2m, 2m+1
    if constexpr (F16X) {
      const uint32_t xw[16] = {Xh[0].x, Xh[0].y, Xh[0].z, Xh[0].w, Xh[1].x, Xh[1].y, Xh[1].z, Xh[1].w,
                               Xh[2].x, Xh[2].y, Xh[2].z, Xh[2].w, Xh[3].x, Xh[3].y, Xh[3].z, Xh[3].w};
#pragma unroll
      for (int m = 0; m < 8; ++m) {                   // xw[i] = (x_2i, x_2i+1); element e of the word at 32c+e
        Bh[m][0] = __byte_perm(xw[m], xw[8 + m], 0x5410);   // (x_2m, x_16+2m)
        Bh[m][1] = __byte_perm(xw[m], xw[8 + m], 0x7632);   // (x_2m+1, x_16+2m+1)
      }
    } else if constexpr (ZB) {
      // B = z (s8) of token gq, bytes ordered like the A slices: Bq[pr][h] byte i = z(32c + 8i + 2pr + h).
      // The 8 plane words X_j (bit e = bit j of z_e) are an 8x8 bit matrix per byte lane; three
      // delta-swap stages transpose it, so register s holds, in byte i, the bits j of element 8i + s.
      uint32_t Z[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) Z[j] = Xz[j];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const uint32_t t = ((Z[j] >> 1) ^ Z[j + 1]) & 0x55555555u;
        Z[j + 1] ^= t;
        Z[j] ^= t << 1;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!(j & 2)) {
          const uint32_t t = ((Z[j] >> 2) ^ Z[j + 2]) & 0x33333333u;
          Z[j + 2] ^= t;
          Z[j] ^= t << 2;
        }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t t = ((Z[j] >> 4) ^ Z[j + 4]) & 0x0F0F0F0Fu;
        Z[j + 4] ^= t;
        Z[j] ^= t << 4;
      }
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        Bq[0][pr][0] = Z[2 * pr];
        Bq[0][pr][1] = Z[2 * pr + 1];
      }
      sxc[0] = sxz[0];
      sxc[1] = sxz[1];
    } else {
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
    }
    // next unit of this warp: band/group, activation prefetch
    int gn = g + 1, bn = b;
    if (gn == NG) { gn = 0; ++bn; }
    int ti0, ti1;
    tiles_of(k, ti0, ti1);
    const bool has_next = k + 1 < n_mine;
    {
      const int gp = has_next ? gn : g;
      if constexpr (F16X) {
        load_xh(gp);
      } else if constexpr (ZB) {
        load_xz(gp);
      } else if constexpr (XQ) {
        const int gi = gp >= xq_g0 ? gp - xq_g0 : gp - xq_g0 + NG;
        Xn[0] = gq < p.l ? s_xq[32 * gi + 4 * gq + c] : 0u;
        sxn[0] = s_xqs[gi];
      } else {
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) {
          Xn[tk] = __ldg(xlane_ptr + ((size_t)tk * NG + gp) * xstride);
          sxn[tk] = __ldg(p.xscales + (size_t)tk * NG + gp);
        }
      }
    }

    uint8_t* sl = ring + slot * Gm::kSlotBytes;
    if (!EXPM(2)) mbar_wait(bars + slot, phase);
    if (k == 0) TSW(1);
    if constexpr (kInitSlots < kSlots) {     // deferred part of the initial fill (in unit order)
      if (k == 0 && lane == 0 && !EXPM(2))
        for (int s2 = kInitSlots; s2 < kSlots && s2 < n_mine; ++s2) issue_next(ring + s2 * Gm::kSlotBytes, bars + s2, s2);
    }

    // tiles are processed two at a time (PT = 2: 4K independent MMA chains hide the IMMA latency); a
    // warp range that starts or ends inside a pair takes that tile alone (PT = 1)
    auto step = [&](auto ptc, const int ib) {
      constexpr int PT = decltype(ptc)::value;

      // lane (gq, c): word c of plane t of rows 16i+gq and 16i+gq+8 (row-major, chunk t at t ^ swz)
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
        if constexpr (IDX) {
          const int x0 = sl[Gm::kPlaneBytes + 16 * i + gq], x1 = sl[Gm::kPlaneBytes + 16 * i + gq + 8];
          const uint2 e0 = reinterpret_cast<const uint2*>(s_tab)[x0], e1 = reinterpret_cast<const uint2*>(s_tab)[x1];
          sb0[j] = e0.x;
          sb1[j] = e1.x;
          r2[j] = make_float2(__uint_as_float(e0.y), __uint_as_float(e1.y));
        } else {
          sb0[j] = *reinterpret_cast<const uint32_t*>(sl + Gm::kPlaneBytes + (16 * i + gq) * 4);
          sb1[j] = *reinterpret_cast<const uint32_t*>(sl + Gm::kPlaneBytes + (16 * i + gq + 8) * 4);
          r2[j] = make_float2(s_rat[sl[Gm::kPlaneBytes + Gm::kSbBytes + 16 * i + gq]],
                              s_rat[sl[Gm::kPlaneBytes + Gm::kSbBytes + 16 * i + gq + 8]]);
        }
      }

      if constexpr (F16X) {
        // ---- fp16-x: M_t = sum_e beta_t[e] x_e on mma.m16n8k16 (fp32 accumulate); K chains of 8 MMAs
        float Df[PT][K][4];
        uint32_t w5[PT][2 * K];
#pragma unroll
        for (int j = 0; j < PT; ++j)
#pragma unroll
          for (int q = 0; q < 2 * K; ++q) w5[j][q] = w[j][q] >> 5;
#pragma unroll
        for (int j = 0; j < PT; ++j)
#pragma unroll
          for (int t = 0; t < K; ++t) Df[j][t][0] = Df[j][t][1] = Df[j][t][2] = Df[j][t][3] = 0.f;
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
          for (int t = 0; t < K; ++t)
#pragma unroll
            for (int j = 0; j < PT; ++j) {
              const uint32_t a0 = f16_bits(w[j][2 * t], w5[j][2 * t], 2 * m);
              const uint32_t a1 = f16_bits(w[j][2 * t + 1], w5[j][2 * t + 1], 2 * m);
              const uint32_t a2 = f16_bits(w[j][2 * t], w5[j][2 * t], 2 * m + 1);
              const uint32_t a3 = f16_bits(w[j][2 * t + 1], w5[j][2 * t + 1], 2 * m + 1);
              mma_f16(Df[j][t], a0, a1, a2, a3, Bh[m][0], Bh[m][1]);
            }
#pragma unroll
        for (int j = 0; j < PT; ++j) {
          const int i = ib + j;
          const float2 s2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] & 0xffffu))),
                                        __half2float(__ushort_as_half((unsigned short)(sb1[j] & 0xffffu))));
          const float2 b2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] >> 16))),
                                        __half2float(__ushort_as_half((unsigned short)(sb1[j] >> 16))));
#pragma unroll
          for (int h = 0; h < 2; ++h) {                 // MMA column 2c+h = token 2c+h; rows (gq, gq+8)
            float2 Ph = make_float2(Df[j][K - 1][h], Df[j][K - 1][2 + h]);
            float2 U = Ph;
#pragma unroll
            for (int t = K - 2; t >= 0; --t) {
              const float2 f = make_float2(Df[j][t][h], Df[j][t][2 + h]);
              Ph = __ffma2_rn(Ph, r2[j], f);
              U = __fadd2_rn(U, f);
            }
            acc[h][i] = __fadd2_rn(acc[h][i], __ffma2_rn(s2, Ph, __fmul2_rn(b2, U)));
          }
        }
        return;
      }

      // ---- AND + popcount on the tensor pipe: PT x K independent chains (tile, plane) of 4 MMAs
      int D[PT][NMMA][K][4];
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        const uint32_t m0 = 0x01010101u << (2 * pr), m1 = 0x01010101u << (2 * pr + 1);
#pragma unroll
        for (int t = 0; t < K; ++t)
#pragma unroll
          for (int j = 0; j < PT; ++j) {
            uint32_t a0, a1, a2, a3;
            if constexpr (ZB) {
              // A bytes are the bits themselves (0/1): shift on the FMA pipe (umulhi), mask on the ALU
              a0 = shr_u(w[j][2 * t], 2 * pr) & 0x01010101u;
              a1 = shr_u(w[j][2 * t + 1], 2 * pr) & 0x01010101u;
              a2 = shr_u(w[j][2 * t], 2 * pr + 1) & 0x01010101u;
              a3 = shr_u(w[j][2 * t + 1], 2 * pr + 1) & 0x01010101u;
            } else {
              a0 = w[j][2 * t] & m0;
              a1 = w[j][2 * t + 1] & m0;
              a2 = w[j][2 * t] & m1;
              a3 = w[j][2 * t + 1] & m1;
            }
#pragma unroll
            for (int tk = 0; tk < NMMA; ++tk) {
              if constexpr (ZB) {
                if (pr == 0)
                  mma_u8s8(D[j][tk][t], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1], 0, 0, 0, 0);
                else
                  mma_u8s8(D[j][tk][t], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1], D[j][tk][t][0], D[j][tk][t][1],
                           D[j][tk][t][2], D[j][tk][t][3]);
              } else {
                if (pr == 0)
                  mma_u8(D[j][tk][t], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1], 0, 0, 0, 0);
                else
                  mma_u8(D[j][tk][t], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1], D[j][tk][t][0], D[j][tk][t][1],
                         D[j][tk][t][2], D[j][tk][t][3]);
              }
            }
          }
      }

#pragma unroll
      for (int j = 0; j < PT; ++j) {
        const int i = ib + j;
        if (DEBUG) {
          const int r0w = 64 * (p.band0 + b) + 16 * i + gq;
#pragma unroll
          for (int t = 0; t < K; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              int32_t* dst = p.P + (((size_t)(r0w + 8 * h) * NG + g) * K + t) * p.l;
              if (j0 < p.l) dst[j0] = D[j][0][t][2 * h] >> 7;
              if (j1 < p.l) dst[j1] = D[j][0][t][2 * h + 1] >> 7;
            }
        } else if constexpr (ZB) {
          // D[j][0][t] = (T_t of rows gq, gq+8) for tokens 2c, 2c+1: sum_e beta_t[e] z_e, exact
          const float2 s2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] & 0xffffu))),
                                        __half2float(__ushort_as_half((unsigned short)(sb1[j] & 0xffffu))));
          const float2 b2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] >> 16))),
                                        __half2float(__ushort_as_half((unsigned short)(sb1[j] >> 16))));
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float2 Ph = __fadd2_rn(make_float2(__int_as_float(imad(D[j][0][K - 1][h], p.one, magic)),
                                               __int_as_float(imad(D[j][0][K - 1][2 + h], p.one, magic))),
                                   make_float2(-cmagic.x, -cmagic.y));
            float2 U = Ph;
#pragma unroll
            for (int t = K - 2; t >= 0; --t) {
              const float2 f = __fadd2_rn(make_float2(__int_as_float(imad(D[j][0][t][h], p.one, magic)),
                                                      __int_as_float(imad(D[j][0][t][2 + h], p.one, magic))),
                                          make_float2(-cmagic.x, -cmagic.y));
              Ph = __ffma2_rn(Ph, r2[j], f);
              U = __fadd2_rn(U, f);
            }
            const float2 v = __ffma2_rn(s2, Ph, __fmul2_rn(b2, U));
            acc[h][i] = __ffma2_rn(make_float2(sxc[h], sxc[h]), v, acc[h][i]);
          }
        } else {
          const float2 s2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] & 0xffffu))),
                                        __half2float(__ushort_as_half((unsigned short)(sb1[j] & 0xffffu))));
          const float2 b2 = make_float2(__half2float(__ushort_as_half((unsigned short)(sb0[j] >> 16))),
                                        __half2float(__ushort_as_half((unsigned short)(sb1[j] >> 16))));
#pragma unroll
          for (int tk = 0; tk < TT; ++tk) {
            // f_t = 128 (P_2c + kappa P_2c+1) for rows (gq, gq+8), exact; Horner over t in fp32x2
            float2 Ph = __fadd2_rn(make_float2(__int_as_float(imad(imad(D[j][tk][K - 1][1], kappa, D[j][tk][K - 1][0]), p.one, magic)),
                                               __int_as_float(imad(imad(D[j][tk][K - 1][3], kappa, D[j][tk][K - 1][2]), p.one, magic))),
                                   make_float2(-cmagic.x, -cmagic.y));
            float2 U = Ph;
#pragma unroll
            for (int t = K - 2; t >= 0; --t) {
              const float2 f = __fadd2_rn(make_float2(__int_as_float(imad(imad(D[j][tk][t][1], kappa, D[j][tk][t][0]), p.one, magic)),
                                                      __int_as_float(imad(imad(D[j][tk][t][3], kappa, D[j][tk][t][2]), p.one, magic))),
                                          make_float2(-cmagic.x, -cmagic.y));
              Ph = __ffma2_rn(Ph, r2[j], f);
              U = __fadd2_rn(U, f);
            }
            const float2 v = __ffma2_rn(s2, Ph, __fmul2_rn(b2, U));
            acc[tk][i] = __ffma2_rn(make_float2(sx[tk], sx[tk]), v, acc[tk][i]);
          }
        }
      }
    };
#pragma unroll
    for (int ib = 0; ib < NB; ib += PTC) {
      if (EXPM(1)) break;
      const bool in0 = ib >= ti0 && ib < ti1;
      if constexpr (PTC == 2) {
        const bool in1 = ib + 1 >= ti0 && ib + 1 < ti1;
        if (in0 && in1) step(std::integral_constant<int, 2>{}, ib);
        else if (in0) step(std::integral_constant<int, 1>{}, ib);
        else if (in1) step(std::integral_constant<int, 1>{}, ib + 1);
      } else {
        if (in0) step(std::integral_constant<int, 1>{}, ib);
      }
    }

    // ---- release the slot and refill it with this warp's unit k + kSlots
    __syncwarp();
    if (lane == 0 && k + kSlots < n_mine && !EXPM(2)) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_next(sl, bars + slot, k + kSlots);
    }
    // this warp has issued its last weight copy: while HBM would drain, pull into L2 the first units that the
    // same warp of the same CTA index fetches first in the next GEMV of the chain (sbvr_gemv_chain)
    if (lane == 0 && p.nx_units && k + kSlots == (n_mine > kSlots ? n_mine : kSlots))
      prefetch_next(p.nx_units, p.nx_NG, p.nx_K, p.nx_C, p.nx_qq, p.nx_rr, cta, wib);
    if (++slot == kSlots) { slot = 0; phase ^= 1u; }

    // ---- leaving band b.  Only a warp's first and last band can be shared with other warps of
    // the CTA, and only a CTA's first and last band with other CTAs.  The warp parks its
    // quad-reduced partial in its smem slot (first / last band); the last warp of the CTA done
    // with the band (smem counter) sums the slots in warp order, then writes y or hands the CTA
    // partial to the band's last CTA.
    if (!DEBUG && (!has_next || bn != b) && !EXPM(4)) {
      // warps of this CTA with tiles in band b: a contiguous run [wf, wl] (ballot over the warps)
      const unsigned int holders =
          __ballot_sync(0xffffffffu, lane < kImmaWarps && s_fb[min(lane, kImmaWarps - 1)] <= b &&
                                         s_lb[min(lane, kImmaWarps - 1)] >= b);
      const int wf = __ffs(holders) - 1, wl = 31 - __clz(holders);
      const bool shared = V0 > b * NG || V1 < min((b + 1) * NG, p.Us);    // other CTAs hold units of b
      float* sp = s_part + ((size_t)wib * 2 + (b == s_fb[wib] ? 0 : 1)) * (TT * 64);
      if constexpr (F16X || ZB) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            const int col = 2 * c + h;                   // token of this MMA column
            if (col < TT) {
              sp[col * 64 + 16 * i + gq] = acc[h][i].x;
              sp[col * 64 + 16 * i + gq + 8] = acc[h][i].y;
            }
            acc[h][i] = make_float2(0.f, 0.f);
          }
      } else {
#pragma unroll
      for (int tk = 0; tk < TT; ++tk)
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          float x0 = acc[tk][i].x * lane_scale, x1 = acc[tk][i].y * lane_scale;
          x0 += __shfl_xor_sync(0xffffffffu, x0, 1);
          x1 += __shfl_xor_sync(0xffffffffu, x1, 1);
          x0 += __shfl_xor_sync(0xffffffffu, x0, 2);
          x1 += __shfl_xor_sync(0xffffffffu, x1, 2);
          if (c == 0) {
            sp[tk * 64 + 16 * i + gq] = x0;
            sp[tk * 64 + 16 * i + gq + 8] = x1;
          }
          acc[tk][i] = make_float2(0.f, 0.f);
        }
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
      TSW(6);
      if (last) {
        __syncwarp();
        __threadfence_block();
        float v[TT][2];
#pragma unroll
        for (int tk = 0; tk < TT; ++tk)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int e = tk * 64 + lane + 32 * h;
            float sum = 0.f;
            for (int w2 = wf; w2 <= wl; ++w2)               // contributing warps, in warp order
              sum += s_part[((size_t)w2 * 2 + (b == s_fb[w2] ? 0 : 1)) * (TT * 64) + e];
            v[tk][h] = sum;
          }
        if (!shared) {
#pragma unroll
          for (int tk = 0; tk < TT; ++tk)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int row = lane + 32 * h;
              if (row < 16 * NB && tk < p.ntok) store_y(p, tk, 64 * (p.band0 + b) + row, v[tk][h]);
            }
        } else {
#if SBVR_MMA_OWNER_PULL
          // owner-pull combine (needs every CTA of the grid co-resident: launched cooperatively)
          if (b == bA && V0 > b * NG) {
            // publisher: band b started in an earlier CTA, whose owner pulls this partial.  Plain
            // stores: every word is self-validating (the slot holds the sentinel until written)
            float* part = p.ws_part + (size_t)cta * 2 * (TT * 64);
#pragma unroll
            for (int tk = 0; tk < TT; ++tk)
#pragma unroll
              for (int h = 0; h < 2; ++h) __stcg(part + tk * 64 + lane + 32 * h, v[tk][h]);
          } else {
            // owner (we hold the band's first unit): pull the later contributors' partials, sum in
            // CTA order, write y, re-arm their slots for the next launch
            const int clast = unit_owner(min((b + 1) * NG, p.Us) - 1, p.qq, p.rr);
            TSW(7);
            for (int cb = cta + 1; cb <= clast; cb += kSumBatch) {
              uint32_t vals[kSumBatch][TT][2];
              // reload the whole batch until no word is the sentinel (a publisher has not written yet):
              // one L2 round trip per poll, not one per stale word
              for (long spins = 0;; ++spins) {
                bool miss = false;
#pragma unroll
                for (int j = 0; j < kSumBatch; ++j)
#pragma unroll
                  for (int tk = 0; tk < TT; ++tk)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                      vals[j][tk][h] = cb + j <= clast
                                           ? ld_relaxed(p.ws_part + (size_t)(cb + j) * 2 * (TT * 64) + tk * 64 + lane + 32 * h)
                                           : 0u;
                      miss |= vals[j][tk][h] == kSentinel;
                    }
                if (!__any_sync(0xffffffffu, miss)) break;
                if (spins > (1L << 24)) __trap();               // a publisher never arrived: fail loudly
              }
#pragma unroll
              for (int j = 0; j < kSumBatch; ++j) {
                if (cb + j > clast) break;
#pragma unroll
                for (int tk = 0; tk < TT; ++tk)
#pragma unroll
                  for (int h = 0; h < 2; ++h) v[tk][h] += __uint_as_float(vals[j][tk][h]);
              }
            }
            for (int c2 = cta + 1; c2 <= clast; ++c2)
#pragma unroll
              for (int tk = 0; tk < TT; ++tk)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  reinterpret_cast<unsigned int*>(p.ws_part)[(size_t)c2 * 2 * (TT * 64) + tk * 64 + lane + 32 * h] = kSentinel;
#pragma unroll
            for (int tk = 0; tk < TT; ++tk)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int row = lane + 32 * h;
                if (row < 16 * NB && tk < p.ntok) store_y(p, tk, 64 * (p.band0 + b) + row, v[tk][h]);
              }
          }
#else
          // band b is shared with other CTAs: last-arriver reduction (no CTA ever waits for another, so
          // nothing depends on the grid being co-resident).  Every contributor stores its CTA partial
          // in its own slot (first / last band of the CTA), fences, and counts itself in on the band's
          // counter; the contributor that arrives last sums ALL slots in CTA order -- the same order
          // whoever arrives last, so y is deterministic -- writes y and re-arms slots and counter.
          // (No memory fence: a fence makes every contributor wait for its stores to be acknowledged
          // before counting itself in.  Instead the reducer validates each word against the at-rest
          // sentinel -- the writers issued those stores before their atomic, so they land in bounded
          // time and the reducer's wait never depends on another CTA making progress.)
          const int myslot = b == bA ? 0 : 1;
          float* part = p.ws_part + ((size_t)cta * 2 + myslot) * (TT * 64);
#pragma unroll
          for (int tk = 0; tk < TT; ++tk)
#pragma unroll
            for (int h = 0; h < 2; ++h) __stcg(part + tk * 64 + lane + 32 * h, v[tk][h]);
          __syncwarp();
          const int c0 = unit_owner(b * NG, p.qq, p.rr);
          const int c1 = unit_owner(min((b + 1) * NG, p.Us) - 1, p.qq, p.rr);
          unsigned int old = 0;
          if (lane == 0) old = atomicAdd(p.ws_cnt + p.band0 + b, 1u);
          old = __shfl_sync(0xffffffffu, old, 0);
          // at rest the counter is 0xFFFFFFFF, so the k-th arrival (k = 1, 2, ...) reads k - 2 (mod 2^32)
          if (old + 2u == (unsigned int)(c1 - c0 + 1)) {
            TSW(7);
            float sum[TT][2];
#pragma unroll
            for (int tk = 0; tk < TT; ++tk) sum[tk][0] = sum[tk][1] = 0.f;
            for (int cb = c0; cb <= c1; cb += kSumBatch) {
              uint32_t vals[kSumBatch][TT][2];
              for (long spins = 0;; ++spins) {       // reload the batch until no word is the sentinel
                bool miss = false;
#pragma unroll
                for (int j = 0; j < kSumBatch; ++j) {
                  const int cc = cb + j;
                  const int fb = (cc * p.qq + min(cc, p.rr)) / NG;          // first band of CTA cc
                  const float* src = p.ws_part + ((size_t)cc * 2 + (b == fb ? 0 : 1)) * (TT * 64);
#pragma unroll
                  for (int tk = 0; tk < TT; ++tk)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                      vals[j][tk][h] = cc > c1 ? 0u : cc == cta ? __float_as_uint(v[tk][h])
                                                                : ld_relaxed(src + tk * 64 + lane + 32 * h);
                      miss |= vals[j][tk][h] == kSentinel;
                    }
                }
                if (!__any_sync(0xffffffffu, miss)) break;
                if (spins > (1L << 26)) __trap();    // stores already issued never landed: fail loudly
              }
#pragma unroll
              for (int j = 0; j < kSumBatch; ++j) {
                if (cb + j > c1) break;
#pragma unroll
                for (int tk = 0; tk < TT; ++tk)
#pragma unroll
                  for (int h = 0; h < 2; ++h) sum[tk][h] += __uint_as_float(vals[j][tk][h]);
              }
            }
            for (int cc = c0; cc <= c1; ++cc) {
              const int fb = (cc * p.qq + min(cc, p.rr)) / NG;
              unsigned int* dst = reinterpret_cast<unsigned int*>(p.ws_part) + ((size_t)cc * 2 + (b == fb ? 0 : 1)) * (TT * 64);
#pragma unroll
              for (int tk = 0; tk < TT; ++tk)
#pragma unroll
                for (int h = 0; h < 2; ++h) dst[tk * 64 + lane + 32 * h] = kSentinel;
            }
            if (lane == 0) p.ws_cnt[p.band0 + b] = kSentinel;
#pragma unroll
            for (int tk = 0; tk < TT; ++tk)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int row = lane + 32 * h;
                if (row < 16 * NB && tk < p.ntok) store_y(p, tk, 64 * (p.band0 + b) + row, sum[tk][h]);
              }
          }
#endif
        }
      }
    }
    if (k + 1 == n_mine) TSW(2);
    b = bn;
    g = gn;
    ++u;
  }
  TSW(3);
#ifdef SBVR_DIAG
  if (p.ts && lane == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.ts[((size_t)blockIdx.x * kImmaWarps + wib) * 8 + 4] = smid;
    p.ts[((size_t)blockIdx.x * kImmaWarps + wib) * 8 + 5] = n_mine;
  }
#endif
}

template <int K, int NB, int TT, bool DEBUG, bool F16X, bool ZB = false, bool IDX = false, bool XQ = false>
inline cudaError_t launch_one(const ImmaParams& p, cudaStream_t st) {
  const int smem = kImmaWarps * Geom<K, NB, IDX>::kWarpBytes + kImmaWarps * 2 * TT * 64 * 4 +
                   (XQ ? p.xq_groups * (32 * 4 + 4) : 0);
  // the attribute is per device; XQ's shared memory grows with the groups per CTA, so keep the largest set
  static int attr_smem[64] = {0};
  const int dev = cur_device();
  if (dev < 0 || dev >= 64 || attr_smem[dev] < smem) {
    cudaError_t e = cudaFuncSetAttribute(gemv_mma_kernel<K, NB, TT, DEBUG, F16X, ZB, IDX, XQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_smem[dev] = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.Pw);
  cfg.blockDim = dim3(kImmaWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[2];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  static const int coop = getenv("SBVR_MMA_COOP") ? atoi(getenv("SBVR_MMA_COOP")) : SBVR_MMA_OWNER_PULL;
  attr_pdl[1].id = cudaLaunchAttributeCooperative;
  attr_pdl[1].val.cooperative = coop;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemv_mma_kernel<K, NB, TT, DEBUG, F16X, ZB, IDX, XQ>, p);
}

template <int K, int NB>
inline cudaError_t launch_nb(const ImmaParams& p, int TT, bool debug, bool f16x, bool zb, cudaStream_t st) {
  if (p.xq) {                              // fp16 x converted in the prologue: batch 1, SBVR-x form, K 2..4
    if constexpr (K >= 2 && K <= 4) {
      if (p.coef_table) return launch_one<K, NB, 1, false, false, false, true, true>(p, st);
      return launch_one<K, NB, 1, false, false, false, false, true>(p, st);
    }
    return cudaErrorInvalidValue;
  }
  if (p.coef_table) {                      // SBVR_META_INDEXED weights: SBVR-x forms, K 2..4 (checked by the ABI)
    if constexpr (K >= 2 && K <= 4) {
      if (zb) return launch_one<K, NB, 8, false, false, true, true>(p, st);
      if (debug) return launch_one<K, NB, 1, true, false, false, true>(p, st);
      if (TT == 1) return launch_one<K, NB, 1, false, false, false, true>(p, st);
      if (TT == 2) return launch_one<K, NB, 2, false, false, false, true>(p, st);
      return launch_one<K, NB, 4, false, false, false, true>(p, st);
    }
    return cudaErrorInvalidValue;
  }
  if (zb) return launch_one<K, NB, 8, false, false, true>(p, st);
  if (f16x) {
    switch (TT) {
      case 1: return launch_one<K, NB, 1, false, true>(p, st);
      case 2: return launch_one<K, NB, 2, false, true>(p, st);
      case 4: return launch_one<K, NB, 4, false, true>(p, st);
      default: return launch_one<K, NB, 8, false, true>(p, st);
    }
  }
  if (debug) return launch_one<K, NB, 1, true, false>(p, st);
  switch (TT) {
    case 1: return launch_one<K, NB, 1, false, false>(p, st);
    case 2: return launch_one<K, NB, 2, false, false>(p, st);
    default: return launch_one<K, NB, 4, false, false>(p, st);
  }
}

template <int K>
cudaError_t launch_k(const ImmaParams& p, int NB, int TT, bool debug, bool f16x, bool zb, cudaStream_t st) {
  switch (NB) {
    case 4: return launch_nb<K, 4>(p, TT, debug, f16x, zb, st);
    case 3: return launch_nb<K, 3>(p, TT, debug, f16x, zb, st);
    case 2: return launch_nb<K, 2>(p, TT, debug, f16x, zb, st);
    default: return launch_nb<K, 1>(p, TT, debug, f16x, zb, st);
  }
}

}  // namespace mma
}  // namespace sbvr
