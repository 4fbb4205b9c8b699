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
// each tile in exactly this lane order, so a warp's 16-byte loads are fully coalesced and land
// in the A registers with no shuffles.
//
// Epilogue per (row, plane): lane c holds columns j = 2c, 2c+1: u = D0 + kappa D1 (exact int),
// with alpha_2c = lane factor folded in at the end; per (row, group):
//     y += s_x * (s * sum_t r^t u_t + b * sum_t u_t)        (c_t = s r^t + b, Eq. 4)
// Rows are reduced over the quad (2 shuffles) only when a warp leaves a band of 64 rows.
//
// Work split: units = (band of 4 row tiles, group) = 4 KB at K = 4, contiguous in memory;
// warp w gets a contiguous unit range (balanced to +-1 unit).  Bands fully inside a warp's
// range are written directly; bands split across warps are combined deterministically by the
// last-arriving warp (integer counter), summing the partial slots in warp order.
#include "sbvr_internal.cuh"

namespace sbvr {

constexpr int kImmaWarps = 8;        // warps per CTA
constexpr int kImmaWarpsPerSM = 16;  // 2 CTAs x 8 warps resident per SM
constexpr int kMaxTT = 4;            // tokens per pass (batched)

struct ImmaParams {
  const uint32_t* planes;
  const uint2* sb2;         // scale_bias as (row gq, row gq+8) pairs
  const uint16_t* ridx2;    // ratio_idx pairs
  const float* ratio_pow;   // [n_ratio][K]
  const uint32_t* xplanes;  // [T][NG][l][4]
  const float* xscales;     // [T][NG]
  float* Y;                 // [T][M]
  int32_t* P;               // debug partials [M][NG][K][l]
  float* ws_part;           // [Pw][2][TT][64]
  unsigned int* ws_cnt;     // [n_bands]
  int M, N, l, n_ratio;
  int Us;                   // units
  int Pw, qq, rr;           // warps and partition
};

__device__ __forceinline__ uint32_t bslice(uint32_t X, int s) {
  // byte b of the result = bit (8b + s) of X placed at bit (7 - s) of byte b
  const int sh = 7 - 2 * s;
  const uint32_t y = sh >= 0 ? (X << sh) : (X >> (-sh));
  return y & (0x01010101u << (7 - s));
}

__device__ __forceinline__ void mma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float lo_half(uint32_t v) {
  return __half2float(__ushort_as_half((unsigned short)(v & 0xffffu)));
}
__device__ __forceinline__ float hi_half(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v >> 16))); }

template <int K>
struct TileRegs {
  uint32_t w[2 * K];  // per plane t: w[2t] = row gq word c, w[2t+1] = row gq+8 word c
  uint2 sb;
  uint32_t ri;
};

template <int K>
__device__ __forceinline__ void load_tile(TileRegs<K>& r, const uint32_t* __restrict__ planes,
                                          const uint2* __restrict__ sb2, const uint16_t* __restrict__ ridx2, long L,
                                          int lane) {
  const uint32_t* base = planes + L * (64L * K);
#pragma unroll
  for (int q = 0; q < K / 2; ++q) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(base + q * 128 + lane * 4));
    r.w[4 * q + 0] = v.x; r.w[4 * q + 1] = v.y; r.w[4 * q + 2] = v.z; r.w[4 * q + 3] = v.w;
  }
  if (K & 1) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(base + (K / 2) * 128 + lane * 2));
    r.w[2 * (K - 1)] = v.x; r.w[2 * (K - 1) + 1] = v.y;
  }
  r.sb = __ldg(sb2 + L * 8 + (lane >> 2));
  r.ri = __ldg(ridx2 + L * 8 + (lane >> 2));
}

__device__ __forceinline__ int unit_owner(int v, int qq, int rr) {
  const int big = rr * (qq + 1);
  return v < big ? v / (qq + 1) : rr + (v - big) / qq;
}

template <int K, int TT, bool DEBUG>
__global__ void __launch_bounds__(kImmaWarps * 32, TT == 1 ? 2 : 1) gemv_imma_kernel(ImmaParams p) {
  __shared__ float s_pow[64 * kMaxK];
  for (int i = threadIdx.x; i < p.n_ratio * K; i += blockDim.x) s_pow[i] = p.ratio_pow[i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * kImmaWarps + (threadIdx.x >> 5);
  if (wid >= p.Pw) return;
  const int gq = lane >> 2, c = lane & 3;
  const int NG = p.N / kG;
  const int MT = p.M / kTileRows;
  const int v0 = wid * p.qq + min(wid, p.rr);
  const int v1 = v0 + p.qq + (wid < p.rr ? 1 : 0);

  // lane constants: columns j0 = 2c, j1 = 2c+1 of the MMA are activation planes; alpha_j = 2^j,
  // alpha_{l-1} = -2^(l-1) (Eq. 12).  u = D0 + kappa*D1 = (alpha_j0 D0 + alpha_j1 D1)/alpha_j0.
  const int j0 = 2 * c, j1 = 2 * c + 1;
  const int al0 = j0 < p.l - 1 ? (1 << j0) : (j0 == p.l - 1 ? -(1 << j0) : 0);
  const int al1 = j1 < p.l - 1 ? (1 << j1) : (j1 == p.l - 1 ? -(1 << j1) : 0);
  const int kappa = al0 != 0 ? al1 / al0 : 0;
  const float lane_scale = (float)al0 * (1.0f / 128.0f);
  const bool xlane = gq < p.l;

  float acc[TT][4][2];
#pragma unroll
  for (int tk = 0; tk < TT; ++tk)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[tk][i][0] = acc[tk][i][1] = 0.0f;

  TileRegs<K> ring[4];
  auto unit_tile0 = [&](int v, int& b, int& g, int& nb) -> long {
    b = v / NG;
    g = v - b * NG;
    nb = min(4, MT - 4 * b);
    return 4L * b * NG + (long)g * nb;
  };
  {
    int b, g, nb;
    const long L0 = unit_tile0(v0, b, g, nb);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < nb) load_tile<K>(ring[i], p.planes, p.sb2, p.ridx2, L0 + i, lane);
  }

  const int first_band = v0 / NG;
  for (int v = v0; v < v1; ++v) {
    int b, g, nb;
    const long L0 = unit_tile0(v, b, g, nb);
    int bn = 0, gn = 0, nbn = 0;
    long Ln = 0;
    const bool has_next = v + 1 < v1;
    if (has_next) Ln = unit_tile0(v + 1, bn, gn, nbn);

    // ---- B operand for group g: activation plane gq, word c, bit-sliced and pre-scaled
    uint32_t Bq[TT][4][2];
    float sx[TT];
#pragma unroll
    for (int tk = 0; tk < TT; ++tk) {
      const uint32_t X = xlane ? __ldg(p.xplanes + ((size_t)tk * NG + g) * (p.l * 4) + gq * 4 + c) : 0u;
      sx[tk] = __ldg(p.xscales + (size_t)tk * NG + g);
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        Bq[tk][pr][0] = bslice(X, 2 * pr);
        Bq[tk][pr][1] = bslice(X, 2 * pr + 1);
      }
    }

#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < nb) {
        const TileRegs<K> tr = ring[i];
        if (has_next && i < nbn) load_tile<K>(ring[i], p.planes, p.sb2, p.ridx2, Ln + i, lane);
        const float* pw0 = s_pow + (tr.ri & 0xffu) * K;
        const float* pw1 = s_pow + (tr.ri >> 8) * K;
        float Pacc[TT][2], Uacc[TT][2];
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) Pacc[tk][0] = Pacc[tk][1] = Uacc[tk][0] = Uacc[tk][1] = 0.0f;
#pragma unroll
        for (int t = 0; t < K; ++t) {
          const uint32_t w0 = tr.w[2 * t], w1 = tr.w[2 * t + 1];
          int D[TT][4];
#pragma unroll
          for (int tk = 0; tk < TT; ++tk) D[tk][0] = D[tk][1] = D[tk][2] = D[tk][3] = 0;
#pragma unroll
          for (int pr = 0; pr < 4; ++pr) {
            const uint32_t m0 = 0x01010101u << (2 * pr), m1 = 0x01010101u << (2 * pr + 1);
            const uint32_t a0 = w0 & m0, a1 = w1 & m0, a2 = w0 & m1, a3 = w1 & m1;
#pragma unroll
            for (int tk = 0; tk < TT; ++tk) mma_u8(D[tk], a0, a1, a2, a3, Bq[tk][pr][0], Bq[tk][pr][1]);
          }
          const float p0 = pw0[t], p1 = pw1[t];
#pragma unroll
          for (int tk = 0; tk < TT; ++tk) {
            const float f0 = (float)(D[tk][0] + kappa * D[tk][1]);
            const float f1 = (float)(D[tk][2] + kappa * D[tk][3]);
            Pacc[tk][0] = fmaf(p0, f0, Pacc[tk][0]);
            Pacc[tk][1] = fmaf(p1, f1, Pacc[tk][1]);
            Uacc[tk][0] += f0;
            Uacc[tk][1] += f1;
          }
          if (DEBUG) {
            const int r0 = 64 * b + 16 * i + gq;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              int32_t* dst = p.P + (((size_t)(r0 + 8 * h) * NG + g) * K + t) * p.l;
              if (j0 < p.l) dst[j0] = D[0][2 * h] >> 7;
              if (j1 < p.l) dst[j1] = D[0][2 * h + 1] >> 7;
            }
          }
        }
        const float s0 = lo_half(tr.sb.x), b0 = hi_half(tr.sb.x);
        const float s1 = lo_half(tr.sb.y), b1 = hi_half(tr.sb.y);
#pragma unroll
        for (int tk = 0; tk < TT; ++tk) {
          acc[tk][i][0] = fmaf(sx[tk], fmaf(s0, Pacc[tk][0], b0 * Uacc[tk][0]), acc[tk][i][0]);
          acc[tk][i][1] = fmaf(sx[tk], fmaf(s1, Pacc[tk][1], b1 * Uacc[tk][1]), acc[tk][i][1]);
        }
      }
    }

    // ---- leaving band b (next unit in another band, or end of range): flush 64 rows
    const bool band_end = !has_next || bn != b;
    if (band_end && !DEBUG) {
      const int band_u0 = b * NG, band_u1 = band_u0 + NG;
      const bool complete = v0 <= band_u0 && band_u1 <= v1;
#pragma unroll
      for (int tk = 0; tk < TT; ++tk)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float x = acc[tk][i][h] * lane_scale;
            x += __shfl_xor_sync(0xffffffffu, x, 1);
            x += __shfl_xor_sync(0xffffffffu, x, 2);
            acc[tk][i][h] = x;
          }
      if (complete) {
        if (c == 0) {
#pragma unroll
          for (int tk = 0; tk < TT; ++tk)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (i < nb) {
                p.Y[(size_t)tk * p.M + 64 * b + 16 * i + gq] = acc[tk][i][0];
                p.Y[(size_t)tk * p.M + 64 * b + 16 * i + gq + 8] = acc[tk][i][1];
              }
        }
      } else {
        const int slot = (b == first_band) ? 0 : 1;
        float* part = p.ws_part + ((size_t)wid * 2 + slot) * (TT * 64);
        if (c == 0) {
#pragma unroll
          for (int tk = 0; tk < TT; ++tk)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              part[tk * 64 + 16 * i + gq] = acc[tk][i][0];
              part[tk * 64 + 16 * i + gq + 8] = acc[tk][i][1];
            }
        }
        __threadfence();
        __syncwarp();
        const int w_lo = unit_owner(band_u0, p.qq, p.rr), w_hi = unit_owner(band_u1 - 1, p.qq, p.rr);
        unsigned int old = 0;
        if (lane == 0) old = atomicAdd(p.ws_cnt + b, 1u);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == (unsigned int)(w_hi - w_lo)) {  // last contributor: combine in warp order
          __threadfence();
          for (int e = lane; e < TT * 64; e += 32) {
            const int tk = e / 64, rr = e % 64;
            float sum = 0.0f;
            for (int w = w_lo; w <= w_hi; ++w) {
              const int wv0 = w * p.qq + min(w, p.rr);
              const int sl = (wv0 / NG == b) ? 0 : 1;
              sum += __ldcg(p.ws_part + ((size_t)w * 2 + sl) * (TT * 64) + e);
            }
            if (16 * (rr / 16) < 16 * nb) p.Y[(size_t)tk * p.M + 64 * b + rr] = sum;
          }
          if (lane == 0) atomicExch(p.ws_cnt + b, 0u);
        }
      }
#pragma unroll
      for (int tk = 0; tk < TT; ++tk)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[tk][i][0] = acc[tk][i][1] = 0.0f;
    }
  }
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
  int Us, Pw, qq, rr, n_bands;
};

static Plan make_plan(const sbvr_weights* w) {
  Plan pl;
  const int NG = w->N / kG, MT = w->M / kTileRows;
  pl.n_bands = (MT + 3) / 4;
  pl.Us = pl.n_bands * NG;
  const int max_warps = num_sms() * kImmaWarpsPerSM;
  pl.Pw = pl.Us < max_warps ? pl.Us : max_warps;
  pl.qq = pl.Us / pl.Pw;
  pl.rr = pl.Us % pl.Pw;
  return pl;
}

size_t imma_workspace_bytes(const sbvr_weights* w, int T) {
  const Plan pl = make_plan(w);
  const int TT = T < kMaxTT ? T : kMaxTT;
  const size_t cnt = ((size_t)pl.n_bands * 4 + 255) / 256 * 256;
  return cnt + (size_t)pl.Pw * 2 * TT * 64 * sizeof(float);
}

template <int K, int TT, bool DEBUG>
static void launch_one(const ImmaParams& p, cudaStream_t st) {
  const int blocks = (p.Pw + kImmaWarps - 1) / kImmaWarps;
  gemv_imma_kernel<K, TT, DEBUG><<<blocks, kImmaWarps * 32, 0, st>>>(p);
}

template <int K>
static void launch_k(const ImmaParams& p, int TT, bool debug, cudaStream_t st) {
  if (debug) { launch_one<K, 1, true>(p, st); return; }
  switch (TT) {
    case 1: launch_one<K, 1, false>(p, st); break;
    case 2: launch_one<K, 2, false>(p, st); break;
    default: launch_one<K, 4, false>(p, st); break;
  }
}

sbvr_status launch_gemv_imma(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                             int32_t* P_debug, cudaStream_t st) {
  const Plan pl = make_plan(w);
  const int NG = w->N / kG;
  ImmaParams p;
  p.planes = w->planes;
  p.sb2 = reinterpret_cast<const uint2*>(w->scale_bias);
  p.ridx2 = reinterpret_cast<const uint16_t*>(w->ratio_idx);
  p.ratio_pow = w->ratio_pow;
  p.M = w->M; p.N = w->N; p.l = x->l; p.n_ratio = w->n_ratio;
  p.Us = pl.Us; p.Pw = pl.Pw; p.qq = pl.qq; p.rr = pl.rr;
  p.P = P_debug;
  const size_t cnt_bytes = ((size_t)pl.n_bands * 4 + 255) / 256 * 256;
  p.ws_cnt = ws ? reinterpret_cast<unsigned int*>(ws) : nullptr;
  p.ws_part = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + cnt_bytes) : nullptr;
  (void)ws_bytes;
  const uint32_t* xp = static_cast<const uint32_t*>(x->data);
  int done = 0;
  while (done < T) {
    const int rem = T - done;
    const int TT = rem >= 4 ? 4 : (rem >= 2 ? 2 : 1);
    p.xplanes = xp + (size_t)done * NG * x->l * 4;
    p.xscales = x->scales + (size_t)done * NG;
    p.Y = Y ? Y + (size_t)done * w->M : nullptr;
    const bool debug = P_debug != nullptr;
    switch (w->K) {
      case 1: launch_k<1>(p, TT, debug, st); break;
      case 2: launch_k<2>(p, TT, debug, st); break;
      case 3: launch_k<3>(p, TT, debug, st); break;
      case 4: launch_k<4>(p, TT, debug, st); break;
      case 5: launch_k<5>(p, TT, debug, st); break;
      case 6: launch_k<6>(p, TT, debug, st); break;
      case 7: launch_k<7>(p, TT, debug, st); break;
      case 8: launch_k<8>(p, TT, debug, st); break;
      default: return set_error(SBVR_ERR_UNSUPPORTED, "K=%d", w->K);
    }
    sbvr_status s = check_launch("gemv_imma_kernel");
    if (s != SBVR_OK) return s;
    if (debug) break;
    done += TT;
  }
  return SBVR_OK;
}

}  // namespace sbvr
