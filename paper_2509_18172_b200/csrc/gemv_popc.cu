// gemv_popc.cu -- the paper's GEMV formulation on CUDA cores (§4.4):
// per (row, group) the inner product of SBVR weights and SBVR activations is
//     sum_t c_t sum_j alpha_j popc(beta_t AND d_j),   c_t = s r^t + b,
// i.e. K*l AND+POPC word pairs per 32 elements and K*l coefficient products per group.
// Kept as the paper-faithful reference kernel (and the partials dump used by the parity
// tests).  On B200 it is POPC-bound: POPC issues at 16 lanes/clk/SM (profiles/r01_step0),
// i.e. ~30% of HBM bandwidth at W4A8 -- the IMMA kernel (gemv_imma.cu) is the fast path.
//
// Mapping: one warp per row, lane over groups (g = lane, lane+32, ...); each lane keeps an
// fp32 partial; fixed-order shuffle reduction; lane 0 writes y.  Activation planes are read
// through the read-only cache (they are reused by every row).
//
// The fp16-x variant (coefficient-weighted sums of fp16 x over the set bits of each plane,
// north star) shares the mapping.
#include "sbvr_internal.cuh"

namespace sbvr {

struct PopcParams {
  const uint8_t* data;
  const float* ratio_pow;
  const uint32_t* xplanes;  // [T][NG][l][4]
  const float* xscales;     // [T][NG]
  float* Y;                 // [T][M] or null
  int32_t* P;               // [M][NG][K][l] or null (debug)
  int M, N, K, l, T;
};

__device__ __forceinline__ float half_lo(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v & 0xffffu))); }
__device__ __forceinline__ float half_hi(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v >> 16))); }

__global__ void __launch_bounds__(256) gemv_popc_kernel(PopcParams p) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= p.M) return;
  const Layout Lo(p.M, p.N, p.K);
  // alpha_j: 2^j for j < l-1, -2^(l-1) for the sign plane (Eq. 12, reading A11)
  for (int tok = 0; tok < p.T; ++tok) {
    float acc = 0.0f;
    for (int g = lane; g < Lo.NG; g += 32) {
      const uint32_t sb = __ldg(reinterpret_cast<const uint32_t*>(p.data + Lo.sb_byte(row, g)));
      const float s = half_lo(sb), b = half_hi(sb);
      const float* pw = p.ratio_pow + (int)__ldg(p.data + Lo.ri_byte(row, g)) * p.K;
      const uint32_t* xp = p.xplanes + ((size_t)tok * Lo.NG + g) * p.l * kWPG;
      float gval = 0.0f;
      for (int t = 0; t < p.K; ++t) {
        uint32_t w[kWPG];
#pragma unroll
        for (int c = 0; c < kWPG; ++c) w[c] = __ldg(reinterpret_cast<const uint32_t*>(p.data + Lo.plane_byte(row, g, t, c)));
        int T_t = 0;
        for (int j = 0; j < p.l; ++j) {
          int P_tj = 0;
#pragma unroll
          for (int c = 0; c < kWPG; ++c) P_tj += __popc(w[c] & __ldg(xp + j * kWPG + c));
          if (p.P) p.P[(((size_t)row * Lo.NG + g) * p.K + t) * p.l + j] = P_tj;
          T_t += (j == p.l - 1) ? -(P_tj << j) : (P_tj << j);
        }
        const float c_t = fmaf(s, __ldg(pw + t), b);
        gval = fmaf(c_t, (float)T_t, gval);
      }
      acc = fmaf(__ldg(p.xscales + (size_t)tok * Lo.NG + g), gval, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && p.Y) p.Y[(size_t)tok * p.M + row] = acc;
  }
}

sbvr_status launch_gemv_popc(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, int32_t* P_debug,
                             cudaStream_t st) {
  PopcParams p;
  p.data = w->data; p.ratio_pow = w->ratio_pow;
  p.xplanes = static_cast<const uint32_t*>(x->data); p.xscales = x->scales;
  p.Y = Y; p.P = P_debug; p.M = w->M; p.N = w->N; p.K = w->K; p.l = x->l; p.T = T;
  const int blocks = (w->M * 32 + 255) / 256;
  gemv_popc_kernel<<<blocks, 256, 0, st>>>(p);
  return check_launch("gemv_popc_kernel");
}

// ------------------------------------------------------------------ fp16-x path (CUDA cores)
// y_r = sum_g sum_t c_t M_t, M_t = sum over set bits e of plane t of x_e (fp32, e ascending).
__global__ void __launch_bounds__(256) gemv_fp16x_kernel(PopcParams p, const uint16_t* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= p.M) return;
  const Layout Lo(p.M, p.N, p.K);
  for (int tok = 0; tok < p.T; ++tok) {
    const uint16_t* xt = x + (size_t)tok * p.N;
    float acc = 0.0f;
    for (int g = lane; g < Lo.NG; g += 32) {
      const uint32_t sb = __ldg(reinterpret_cast<const uint32_t*>(p.data + Lo.sb_byte(row, g)));
      const float s = half_lo(sb), b = half_hi(sb);
      const float* pw = p.ratio_pow + (int)__ldg(p.data + Lo.ri_byte(row, g)) * p.K;
      float gval = 0.0f;
      for (int t = 0; t < p.K; ++t) {
        float M_t = 0.0f;
        for (int c = 0; c < kWPG; ++c) {
          uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(p.data + Lo.plane_byte(row, g, t, c)));
          while (w) {
            const int e = __ffs(w) - 1;
            w &= w - 1;
            M_t += __half2float(__ushort_as_half(__ldg(xt + g * kG + 32 * c + e)));
          }
        }
        gval = fmaf(fmaf(s, __ldg(pw + t), b), M_t, gval);
      }
      acc += gval;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) p.Y[(size_t)tok * p.M + row] = acc;
  }
}

sbvr_status launch_gemv_fp16x(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, cudaStream_t st) {
  PopcParams p;
  p.data = w->data; p.ratio_pow = w->ratio_pow;
  p.xplanes = nullptr; p.xscales = nullptr;
  p.Y = Y; p.P = nullptr; p.M = w->M; p.N = w->N; p.K = w->K; p.l = 0; p.T = T;
  const int blocks = (w->M * 32 + 255) / 256;
  gemv_fp16x_kernel<<<blocks, 256, 0, st>>>(p, static_cast<const uint16_t*>(x->data));
  return check_launch("gemv_fp16x_kernel");
}

}  // namespace sbvr
