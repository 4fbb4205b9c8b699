// gemv_tc.cu -- SBVR GEMV (§4.4) with the AND+popcount inner products on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in tensor memory).
//
// Per (row, group, weight plane t, activation plane j) the paper needs P_tj = popc(beta_t AND d_j)
// and then y_row += s_x * sum_t c_t sum_j alpha_j P_tj with c_t = s r^t + b (Eq. 4, Eq. 12).
// A u8 MMA whose operands are single bits IS an AND+popcount:
//     A[row][k] = bit(beta_t, e(k)) * 2^s      (one LOP3: plane_word & (0x01010101 << s))
//     B[k][j]   = bit(d_j,   e(k)) * 2^(7-s)   (activation plane j, bit-sliced once per group)
// so every product is 128 * (beta AND d) and D[row][j] summed over a group's 128 elements is
// exactly 128 * P_tj.  Element e(k) of MMA chunk q (32 elements = plane word q) at k = 4s + b is
// bit 8b + s of word q.
//
// Kernel shape (one CTA per SM, persistent over a balanced contiguous range of units):
//   unit = (row block of 128 rows, group) = 128 x K plane words + scale/bias + ratio index,
//          streamed global -> shared by TMA bulk copies (cp.async.bulk, mbarrier complete_tx)
//   worker group (4 warps, thread = row = TMEM lane):
//          LDS.128 per plane -> 32 LOP3 -> tcgen05.st.32x32b.x32 into the group's A region of
//          tensor memory; the 4 bit-sliced activation matrices B_q [8 planes][32 k] go to smem
//   control warp (one elected thread): K x 4 tcgen05.mma M=128 N=8*TT K=32 per unit, A from
//          TMEM, B from smem (K-major canonical, no swizzle), D (s32) in TMEM; tcgen05.commit
//          -> mbarrier; refills the TMA ring
//   epilogue (same worker thread): tcgen05.ld of its row's K x 8 s32 accumulators,
//          T_t = sum_j alpha_j D_tj (IMAD), exact int->float via the 1.5*2^23 magic number,
//          Horner sum_t r^t T_t, y += s_x (s * that + b * sum_t T_t)
// Two or three worker groups alternate units so one group's LOP3/tcgen05.st phase overlaps the
// other's MMA latency and epilogue.  Row blocks split across CTAs are combined deterministically:
// the first contributor (owner) adds the partials the later contributors published (release
// flags), in (CTA, group) order.
#include <cstdlib>

#include "sbvr_internal.cuh"

namespace sbvr {

constexpr int kTcSlots = 4;      // TMA ring depth (units)
constexpr int kMaxTT = 4;        // tokens per pass (batched)
constexpr int kRbPerCta = 6;     // row blocks a CTA range may touch (host guarantees)
constexpr int kMaxPre = 8;       // later CTAs sharing the owner's last row block (host guarantees)
constexpr int kMaxGroups = 3;    // worker groups

struct TcParams {
  const uint8_t* units;     // packed unit records (sbvr.h layout)
  const float* ratio_pow;   // [n_ratio][K]
  const uint32_t* xplanes;  // [T][NG][l][4]
  const float* xscales;     // [T][NG]
  float* Y;                 // [T][M]
  int32_t* P;               // debug partials [M][NG][K][l]
  float* ws_part;           // [C][group][TT][128] partials of each CTA's first row block when shared
  unsigned int* ws_cnt;     // [C][group] publish flags: 1 = set by the publisher, 0xFFFFFFFF = cleared (owner)
  int M, N, l, n_ratio;
  int n_full, tail_rows;    // full row blocks, rows of the tail block (0 if none)
  int Us;                   // units
  int C, qq, rr;            // CTAs and the unit partition over CTAs
  int one;                  // = 1 (runtime value, see i2f_fma)
  int exp_mode;             // ablation bits (env SBVR_EXP_MODE, 0 in production): 1 skip MMAs,
                            // 2 skip the A build, 4 skip the epilogue, 8 phase timestamps
  unsigned long long* ts;   // [C][8] globaltimer stamps (exp_mode & 8, env SBVR_TS_PTR)
};
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TS(slot) do { if (p.exp_mode & 8) p.ts[(size_t)blockIdx.x * 32 + (slot)] = gtime(); } while (0)

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
// wait for outstanding tcgen05.ld; every loaded register is then threaded through an empty
// volatile asm so no use of it can be hoisted above the wait
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void pin8(uint32_t (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) asm volatile("" : "+r"(v[i]));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_i8(uint32_t tD, uint32_t tA, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
      "r"(tA), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8 rows x 16 bytes,
// LBO = byte distance between the two 16-element K halves, SBO = between 8-row groups
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ uint32_t bslice(uint32_t X, int s) {
  // byte b of the result = bit (8b + s) of X placed at bit (7 - s) of byte b
  const int sh = 7 - 2 * s;
  const uint32_t y = sh >= 0 ? (X << sh) : (X >> (-sh));
  return y & (0x01010101u << (7 - s));
}

// exact int -> float for |u| < 2^22 on the FMA pipe: (u + 0x4B400000) as float - 1.5*2^23
__device__ __forceinline__ float i2f_fma(int u, int one) {
  int v;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(v) : "r"(u), "r"(one), "r"(0x4B400000));
  return __int_as_float(v) - 12582912.0f;
}

__device__ __forceinline__ int unit_owner(int v, int qq, int rr) {
  const int big = rr * (qq + 1);
  return v < big ? v / (qq + 1) : rr + (v - big) / qq;
}

template <int K>
struct TcGeom {
  static constexpr int kUnitFull = 128 * (16 * K + 5);                // bytes of a full-block unit
  static constexpr int kSlotBytes = (kUnitFull + 127) / 128 * 128;
  static constexpr int kACols = 32 * K;                               // TMEM columns of A per group
};

template <int K, int TT, int NWG, bool DEBUG>
__global__ void __launch_bounds__(NWG * 128 + 32, 1) gemv_tc_kernel(TcParams p) {
  using Gm = TcGeom<K>;
  constexpr int kDCols = 8 * TT * K;                 // TMEM columns of D per group
  constexpr int kBBytes = 4 * 256 * TT;              // B_q matrices of one unit
  constexpr int kWorkers = NWG * 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  // dynamic smem: [ring: kTcSlots x slot][B: NWG x kBBytes][s_part: kRbPerCta x NWG x TT x 128]
  //               [s_pre: kMaxPre x NWG x TT x 128]
  uint8_t* ring = smem;
  uint8_t* sB = smem + kTcSlots * Gm::kSlotBytes;
  float* s_part = reinterpret_cast<float*>(sB + NWG * kBBytes);
  float* s_pre = s_part + kRbPerCta * NWG * TT * 128;
  __shared__ float s_rat[64];
  __shared__ __align__(8) uint64_t bar_full[kTcSlots];
  __shared__ __align__(8) uint64_t bar_a[kMaxGroups];
  __shared__ __align__(8) uint64_t bar_d[kMaxGroups];
  __shared__ uint32_t s_tmem;

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) TS(0);
  const int NG = p.N / kG;
  const int cta = blockIdx.x;
  const int V0 = cta * p.qq + min(cta, p.rr);
  const int V1 = V0 + p.qq + (cta < p.rr ? 1 : 0);
  const int n = V1 - V0;
  const long full_units = (long)p.n_full * NG;
  auto unit_src = [&](int u) -> const uint8_t* {
    return u < full_units ? p.units + (size_t)u * Gm::kUnitFull
                          : p.units + (size_t)full_units * Gm::kUnitFull +
                                (size_t)(u - full_units) * (p.tail_rows * (16 * K + 5));
  };
  auto unit_bytes = [&](int u) -> uint32_t {
    return u < full_units ? (uint32_t)Gm::kUnitFull : (uint32_t)(p.tail_rows * (16 * K + 5));
  };

  if (warp == NWG * 4) {
    // control warp: TMEM allocation, barriers, first TMA copies (weights are immutable, so they
    // may start before the previous kernel finishes: programmatic dependent launch)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) {
      for (int s = 0; s < kTcSlots; ++s) mbar_init(&bar_full[s], 1);
      for (int g = 0; g < NWG; ++g) {
        mbar_init(&bar_a[g], 128);
        mbar_init(&bar_d[g], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int s = 0; s < kTcSlots && s < n; ++s) {
        mbar_expect_tx(&bar_full[s], unit_bytes(V0 + s));
        bulk_g2s(ring + s * Gm::kSlotBytes, unit_src(V0 + s), unit_bytes(V0 + s), &bar_full[s]);
      }
    }
  }
  for (int i = tid; i < p.n_ratio; i += blockDim.x) s_rat[i] = K >= 2 ? p.ratio_pow[i * K + 1] : 0.f;
  for (int i = tid; i < kRbPerCta * NWG * TT * 128; i += blockDim.x) s_part[i] = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tid == 0) TS(1);

  const int rbA = V0 / NG, rbZ = (V1 - 1) / NG;
  const bool pubA = V0 > rbA * NG;                                   // rbA started in an earlier CTA
  const bool ownZ = V1 < (rbZ + 1) * NG && !(rbZ == rbA && pubA);    // we hold rbZ's first unit
  const int c_hiZ = ownZ ? unit_owner((rbZ + 1) * NG - 1, p.qq, p.rr) : cta;
  const int nPre = ownZ ? (c_hiZ - cta) * NWG : 0;                   // (CTA, group) slots to add

  if (warp == NWG * 4) {
    // ---------------------------------------------------------------- MMA issue + TMA refill
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | ((uint32_t)(8 * TT / 8) << 17) | (8u << 24);  // s32 += u8*u8, N=8TT, M=128
      for (int k = 0; k < n; ++k) {
        const int grp = k % NWG, it = k / NWG;
        mbar_wait(&bar_a[grp], it & 1);
        tc_fence_after();
        if (k < 6) TS(5 + k);
        const uint32_t tA = tmem + grp * Gm::kACols;
        const uint32_t tD = tmem + NWG * Gm::kACols + grp * kDCols;
        const uint32_t bbase = smem_u32(sB + grp * kBBytes);
        if (!(p.exp_mode & 1))
#pragma unroll
        for (int t = 0; t < K; ++t)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mma_i8(tD + 8 * TT * t, tA + 32 * t + 8 * q, smem_desc(bbase + q * 256 * TT, 128, 256), idesc, q);
        mma_commit(&bar_d[grp]);
        // the workers arrived on bar_a after reading unit k's slot: refill it with unit k + slots
        if (k + kTcSlots < n) {
          const int s = k % kTcSlots;
          mbar_expect_tx(&bar_full[s], unit_bytes(V0 + k + kTcSlots));
          bulk_g2s(ring + s * Gm::kSlotBytes, unit_src(V0 + k + kTcSlots), unit_bytes(V0 + k + kTcSlots),
                   &bar_full[s]);
        }
      }
      TS(3);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- worker groups
    const int grp = warp >> 2, r = tid & 127;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t tA = tmem + lane_base + grp * Gm::kACols;
    const uint32_t tD = tmem + lane_base + NWG * Gm::kACols + grp * kDCols;
    uint8_t* myB = sB + grp * kBBytes;
    const int sw = chunk_swizzle(K, r);
    // Eq. 12 plane weights: alpha_j = 2^j (j < l-1), alpha_{l-1} = -2^(l-1), 0 beyond l
    int alpha[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) alpha[j] = j < p.l - 1 ? (1 << j) : (j == p.l - 1 ? -(1 << j) : 0);
    const int one = p.one;

    // activation words for the B matrices of a unit: thread r builds words idx = r + 128 e
    // (idx -> q = idx / (64 TT), n = (idx / 8) % (8 TT) = 8 tk + j, s = idx % 8)
    auto load_x = [&](int g, uint32_t (&X)[2 * TT], float (&sx)[TT]) {
#pragma unroll
      for (int e = 0; e < 2 * TT; ++e) {
        const int idx = r + 128 * e;
        const int q = idx / (64 * TT), nn = (idx >> 3) % (8 * TT), tk = nn >> 3, j = nn & 7;
        X[e] = j < p.l ? __ldg(p.xplanes + (((size_t)tk * NG + g) * p.l + j) * 4 + q) : 0u;
      }
#pragma unroll
      for (int tk = 0; tk < TT; ++tk) sx[tk] = __ldg(p.xscales + (size_t)tk * NG + g);
    };

    float acc[TT];
#pragma unroll
    for (int tk = 0; tk < TT; ++tk) acc[tk] = 0.f;
    int cur_rb = -1;
    bool published = false;
    uint32_t Xn[2 * TT];
    float sxn[TT];
    if (grp < n) load_x((V0 + grp) % NG, Xn, sxn);

    auto flush = [&](int rb) {
      // leaving row block rb: park the partial in smem, or publish it if rb is shared with an
      // earlier CTA (its owner adds it)
      if (rb == rbA && pubA) {
        float* dst = p.ws_part + ((size_t)cta * NWG + grp) * (TT * 128);
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) dst[tk * 128 + r] = acc[tk];
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
        if (r == 0)
          asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(p.ws_cnt + cta * NWG + grp) : "memory");
        published = true;
      } else {
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) s_part[(((rb - rbA) * NWG + grp) * TT + tk) * 128 + r] = acc[tk];
      }
#pragma unroll
      for (int tk = 0; tk < TT; ++tk) acc[tk] = 0.f;
    };

    for (int k = grp; k < n; k += NWG) {
      const int it = k / NWG;
      const int u = V0 + k;
      const int rb = u / NG, g = u - rb * NG;
      const int rows = rb < p.n_full ? 128 : p.tail_rows;
      if (!DEBUG && rb != cur_rb) {
        if (cur_rb >= 0) flush(cur_rb);
        cur_rb = rb;
      }
      uint32_t X[2 * TT];
      float sx[TT];
#pragma unroll
      for (int e = 0; e < 2 * TT; ++e) X[e] = Xn[e];
#pragma unroll
      for (int tk = 0; tk < TT; ++tk) sx[tk] = sxn[tk];
      if (k + NWG < n) load_x((V0 + k + NWG) % NG, Xn, sxn);

      // ---- B_q [8 TT n][32 k] for this unit's group (the previous MMA reading myB has completed:
      // we waited for its commit before the previous epilogue)
#pragma unroll
      for (int e = 0; e < 2 * TT; ++e) {
        const int idx = r + 128 * e;
        const int q = idx / (64 * TT), nn = (idx >> 3) % (8 * TT), s = idx & 7;
        const uint32_t v = bslice(X[e], s);
        *reinterpret_cast<uint32_t*>(myB + q * 256 * TT + (nn >> 3) * 256 + (s >> 2) * 128 + (nn & 7) * 16 +
                                     (s & 3) * 4) = v;
      }

      // ---- A: this thread's row, K planes x 32 masked words -> TMEM
      const int slot = k % kTcSlots;
      mbar_wait(&bar_full[slot], (k / kTcSlots) & 1);
      if (tid == 0 && it < 4) TS(12 + it);
      const uint8_t* sl = ring + slot * Gm::kSlotBytes;
      const bool valid = r < rows;
      if (!(p.exp_mode & 2))
#pragma unroll
      for (int t = 0; t < K; ++t) {
        uint4 w4 = make_uint4(0u, 0u, 0u, 0u);
        if (valid) w4 = *reinterpret_cast<const uint4*>(sl + r * 16 * K + 16 * (t ^ sw));
        uint32_t a[32];
        const uint32_t wq[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int s = 0; s < 8; ++s) a[8 * q + s] = wq[q] & (0x01010101u << s);
        tmem_st32(tA + 32 * t, a);
      }
      uint32_t sbw = 0, ri = 0;
      if (valid) {
        sbw = *reinterpret_cast<const uint32_t*>(sl + rows * 16 * K + 4 * r);
        ri = sl[rows * (16 * K + 4) + r];
      }
      tmem_wait_st();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // B (generic stores) -> MMA (async proxy)
      tc_fence_before();
      mbar_arrive(&bar_a[grp]);

      // ---- epilogue: wait for this unit's MMAs, read the row's accumulators
      mbar_wait(&bar_d[grp], it & 1);
      tc_fence_after();
      if (tid == 0 && it < 4) TS(16 + it);
      if (DEBUG) {
#pragma unroll
        for (int t = 0; t < K; ++t) {
          uint32_t d[8];
          tmem_ld8(tD + 8 * TT * t, d);
          tmem_wait_ld();
          pin8(d);
          if (valid) {
            const int row = rb * 128 + r;
            int32_t* dst = p.P + (((size_t)row * NG + g) * K + t) * p.l;
            for (int j = 0; j < p.l; ++j) dst[j] = (int32_t)d[j] >> 7;
          }
        }
        continue;
      }
      if (p.exp_mode & 4) continue;
      const float s_ = __half2float(__ushort_as_half((unsigned short)(sbw & 0xffffu)));
      const float b_ = __half2float(__ushort_as_half((unsigned short)(sbw >> 16)));
      const float rr_ = s_rat[ri];
#pragma unroll
      for (int tk = 0; tk < TT; ++tk) {
        uint32_t d[K][8];
#pragma unroll
        for (int t = 0; t < K; ++t) tmem_ld8(tD + 8 * TT * t + 8 * tk, d[t]);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < K; ++t) pin8(d[t]);
        float Ph = 0.f, U = 0.f;
#pragma unroll
        for (int t = K - 1; t >= 0; --t) {
          int T = (int)d[t][0] * alpha[0];
#pragma unroll
          for (int j = 1; j < 8; ++j) T += (int)d[t][j] * alpha[j];
          const float f = i2f_fma(T, one);      // = 128 * sum_j alpha_j P_tj, exact
          Ph = (t == K - 1) ? f : fmaf(Ph, rr_, f);
          U += f;
        }
        acc[tk] = fmaf(sx[tk], fmaf(s_, Ph, b_ * U), acc[tk]);
      }
      if (tid == 0 && it < 4) TS(20 + it);
    }
    if (tid == 0) TS(2);
    if (!DEBUG) {
      if (cur_rb >= 0) flush(cur_rb);
      // a group with no unit in the shared first row block still publishes (zeros) so the
      // owner's wait ends
      if (pubA && !published) {
        float* dst = p.ws_part + ((size_t)cta * NWG + grp) * (TT * 128);
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) dst[tk * 128 + r] = 0.f;
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
        if (r == 0)
          asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(p.ws_cnt + cta * NWG + grp) : "memory");
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == NWG * 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
  if (DEBUG) return;

  // ---- owner of rbZ: acquire the later contributors' flags, stage their partials in smem
  if (nPre > 0) {
    for (int q = tid; q < nPre; q += blockDim.x) {
      unsigned int f = 0;
      long spins = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(p.ws_cnt + (cta + 1) * NWG + q) : "memory");
        if (++spins > (1L << 28)) __trap();     // a publisher never arrived: fail loudly, never hang
      } while (f != 1u);
    }
    __syncthreads();
    const float* src = p.ws_part + ((size_t)(cta + 1) * NWG) * (TT * 128);
    for (int e = tid; e < nPre * TT * 128; e += blockDim.x) s_pre[e] = __ldcg(src + e);
    __syncthreads();
    // back to rest (all 0xFF, sbvr_workspace_init): the workspace may be shared with kernels whose slots
    // are sentinel-validated (PIPE)
    for (int e = tid; e < nPre * TT * 128; e += blockDim.x)
      reinterpret_cast<unsigned int*>(const_cast<float*>(src))[e] = 0xFFFFFFFFu;
    for (int q = tid; q < nPre; q += blockDim.x) p.ws_cnt[(cta + 1) * NWG + q] = 0xFFFFFFFFu;   // reset for the next launch
  }
  // ---- CTA combine in (group) order; row blocks we published are finished by their owner
  const int nrb = rbZ - rbA + 1;
  for (int e = tid; e < nrb * TT * 128; e += blockDim.x) {
    const int bl = e / (TT * 128), tk = (e / 128) % TT, row = e % 128;
    const int rb = rbA + bl;
    const int rows = rb < p.n_full ? 128 : p.tail_rows;
    if (row >= rows || (rb == rbA && pubA)) continue;
    float sum = 0.f;
#pragma unroll
    for (int g2 = 0; g2 < NWG; ++g2) sum += s_part[((bl * NWG + g2) * TT + tk) * 128 + row];
    if (rb == rbZ && ownZ)
      for (int q = 0; q < nPre; ++q) sum += s_pre[(q * TT + tk) * 128 + row];
    p.Y[(size_t)tk * p.M + (size_t)rb * 128 + row] = sum * (1.0f / 128.0f);
  }
  if (tid == 0) TS(4);
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

// worker groups: as many as tensor memory holds (A + D per group <= 512 columns), at most 3
static int groups_for(int K, int TT) {
  const int per = 32 * K + 8 * TT * K;
  int g = 512 / per;
  if (g > kMaxGroups) g = kMaxGroups;
  return g;
}

struct TcPlan {
  int NG, n_full, tail_rows, n_rb, Us, C;
};

// one CTA per SM, but enough CTAs that a range touches <= kRbPerCta row blocks, few enough that a
// row block is shared by <= kMaxPre + 1 CTAs, never more CTAs than units
static TcPlan make_plan(const sbvr_weights* w) {
  TcPlan pl;
  pl.NG = w->N / kG;
  pl.n_full = w->M / kRowBlock;
  pl.tail_rows = w->M % kRowBlock;
  pl.n_rb = pl.n_full + (pl.tail_rows ? 1 : 0);
  pl.Us = pl.n_rb * pl.NG;
  int C = num_sms();
  const int max_range = (kRbPerCta - 1) * pl.NG;
  const int need = (pl.Us + max_range - 1) / max_range + 1;
  if (C < need) C = need;
  const int min_range = (pl.NG + kMaxPre - 1) / kMaxPre;
  const int cap = pl.Us / min_range;
  if (C > cap && cap >= 1) C = cap;
  if (C > pl.Us) C = pl.Us;
  if (C < 1) C = 1;
  pl.C = C;
  return pl;
}

size_t tc_workspace_bytes(const sbvr_weights* w, int T) {
  const TcPlan pl = make_plan(w);
  const int TT = T < kMaxTT ? T : kMaxTT;
  const size_t flags = ((size_t)pl.C * kMaxGroups * 4 + 255) / 256 * 256;
  return flags + (size_t)pl.C * kMaxGroups * TT * 128 * sizeof(float);
}

template <int K, int TT, int NWG, bool DEBUG>
static cudaError_t launch_one(const TcParams& p, cudaStream_t st) {
  constexpr int kBBytes = 4 * 256 * TT;
  const int smem = kTcSlots * TcGeom<K>::kSlotBytes + NWG * kBBytes + (kRbPerCta + kMaxPre) * NWG * TT * 128 * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(gemv_tc_kernel<K, TT, NWG, DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.C);
  cfg.blockDim = dim3(NWG * 128 + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemv_tc_kernel<K, TT, NWG, DEBUG>, p);
}

template <int K, int TT, bool DEBUG>
static cudaError_t launch_g(const TcParams& p, cudaStream_t st) {
  constexpr int per = 32 * K + 8 * TT * K;
  constexpr int G0 = 512 / per;
  constexpr int NWG = G0 > kMaxGroups ? kMaxGroups : G0;
  static_assert(NWG >= 1, "tensor memory too small");
  return launch_one<K, TT, NWG, DEBUG>(p, st);
}

template <int K>
static cudaError_t launch_k(const TcParams& p, int TT, bool debug, cudaStream_t st) {
  if (debug) return launch_g<K, 1, true>(p, st);
  switch (TT) {
    case 1: return launch_g<K, 1, false>(p, st);
    case 2: return launch_g<K, 2, false>(p, st);
    default: return launch_g<K, 4, false>(p, st);
  }
}

static cudaError_t launch_any(int K, const TcParams& p, int TT, bool debug, cudaStream_t st) {
  switch (K) {
    case 1: return launch_k<1>(p, TT, debug, st);
    case 2: return launch_k<2>(p, TT, debug, st);
    case 3: return launch_k<3>(p, TT, debug, st);
    case 4: return launch_k<4>(p, TT, debug, st);
    case 5: return launch_k<5>(p, TT, debug, st);
    case 6: return launch_k<6>(p, TT, debug, st);
    case 7: return launch_k<7>(p, TT, debug, st);
    default: return launch_k<8>(p, TT, debug, st);
  }
}

sbvr_status launch_gemv_tc(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                           int32_t* P_debug, cudaStream_t st) {
  const TcPlan pl = make_plan(w);
  // the owner/publisher fix-up needs every CTA resident at once (one CTA per SM)
  if (pl.C > num_sms())
    return set_error(SBVR_ERR_UNSUPPORTED, "M=%d N=%d needs %d CTAs > %d SMs", w->M, w->N, pl.C, num_sms());
  TcParams p;
  p.units = w->data;
  p.ratio_pow = w->ratio_pow;
  p.M = w->M; p.N = w->N; p.l = x->l; p.n_ratio = w->n_ratio;
  p.n_full = pl.n_full;
  p.tail_rows = pl.tail_rows;
  p.Us = pl.Us;
  p.C = pl.C;
  p.qq = pl.Us / pl.C;
  p.rr = pl.Us % pl.C;
  p.P = P_debug;
  p.one = 1;
  {
    const char* em = getenv("SBVR_EXP_MODE");
    p.exp_mode = em ? atoi(em) : 0;
    const char* tsp = getenv("SBVR_TS_PTR");
    p.ts = tsp ? reinterpret_cast<unsigned long long*>(strtoull(tsp, nullptr, 0)) : nullptr;
    if (!p.ts) p.exp_mode &= ~8;
  }
  const size_t cnt_bytes = ((size_t)pl.C * kMaxGroups * 4 + 255) / 256 * 256;
  p.ws_cnt = ws ? reinterpret_cast<unsigned int*>(ws) : nullptr;
  p.ws_part = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + cnt_bytes) : nullptr;
  (void)ws_bytes;
  const uint32_t* xp = static_cast<const uint32_t*>(x->data);
  const bool debug = P_debug != nullptr;
  int done = 0;
  while (done < T) {
    const int rem = T - done;
    int TT = debug ? 1 : (rem >= 4 ? 4 : (rem >= 2 ? 2 : 1));
    while (TT > 1 && groups_for(w->K, TT) < 1) TT >>= 1;
    p.xplanes = xp + (size_t)done * pl.NG * x->l * 4;
    p.xscales = x->scales + (size_t)done * pl.NG;
    p.Y = Y ? Y + (size_t)done * w->M : nullptr;
    cudaError_t e = launch_any(w->K, p, TT, debug, st);
    if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "gemv_tc setup: %s", cudaGetErrorString(e));
    sbvr_status s = check_launch("gemv_tc_kernel");
    if (s != SBVR_OK) return s;
    if (debug) break;
    done += TT;
  }
  return SBVR_OK;
}

}  // namespace sbvr
