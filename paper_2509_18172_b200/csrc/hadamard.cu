// hadamard.cu -- randomized Hadamard rotation, PAPER.md P:255 (§4.5): weights are rotated before SBVR
// encoding to Gaussianize them and suppress outliers (and activations by the same orthogonal Q at run
// time, so y = (W Q^T)(Q x)).  Reading A21: block-diagonal along N, blocks of b = 2^k
// columns, Q = H_b diag(signs) / sqrt(b), H_b[i][k] = (-1)^popcount(i & k) (Sylvester order).
//
// One warp per (row, block), b in [32, 1024]: lane L holds elements L + 32 i (i < b/32), so the loads
// and stores are coalesced 128-byte rows.  The fast Walsh-Hadamard transform runs the log2(b)
// butterflies (a, c) -> (a + c, a - c) on index bit h: bits 0-4 (the lane) with __shfl_xor_sync,
// bits >= 5 inside the lane's registers.  fp32 arithmetic; fp32 or fp16 in/out; in place allowed
// (a warp reads its whole block before writing).  HBM-bound: 2 x element bytes per element.
#include "sbvr_internal.cuh"

namespace sbvr {
namespace {

template <int M, bool HALF>
__global__ void __launch_bounds__(256) hadamard_kernel(const void* X, void* Y, const int8_t* __restrict__ signs,
                                                       long n_blocks, int N, float scale) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int B = 32 * M;
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * (blockDim.x >> 5);
  const int nb = N / B;
  for (long q = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n_blocks; q += warps) {
    const long row = q / nb;
    const int blk = (int)(q - row * nb);
    const size_t base = (size_t)row * N + (size_t)blk * B;
    float v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int e = lane + 32 * i;
      const float x = HALF ? __half2float(reinterpret_cast<const __half*>(X)[base + e])
                           : reinterpret_cast<const float*>(X)[base + e];
      v[i] = signs[(size_t)blk * B + e] < 0 ? -x : x;
    }
    // index bits >= 5: in registers
#pragma unroll
    for (int h = 1; h < M; h <<= 1)
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (!(i & h)) {
          const float a = v[i], c = v[i + h];
          v[i] = a + c;
          v[i + h] = a - c;
        }
    // index bits 0-4: across lanes
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
      const bool hi = lane & h;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const float o = __shfl_xor_sync(0xffffffffu, v[i], h);
        v[i] = hi ? o - v[i] : v[i] + o;
      }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int e = lane + 32 * i;
      const float y = v[i] * scale;
      if (HALF) reinterpret_cast<__half*>(Y)[base + e] = __float2half_rn(y);
      else reinterpret_cast<float*>(Y)[base + e] = y;
    }
  }
}

template <bool HALF>
static cudaError_t launch_h(int b, const void* X, void* Y, const int8_t* signs, long n_blocks, int N, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long want = (n_blocks + 7) / 8;
  const int grid = (int)std::min<long>(want, (long)sms * 8);
  const float scale = (float)(1.0 / sqrt((double)b));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid > 0 ? grid : 1);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (b) {
    case 32: return cudaLaunchKernelEx(&cfg, hadamard_kernel<1, HALF>, X, Y, signs, n_blocks, N, scale);
    case 64: return cudaLaunchKernelEx(&cfg, hadamard_kernel<2, HALF>, X, Y, signs, n_blocks, N, scale);
    case 128: return cudaLaunchKernelEx(&cfg, hadamard_kernel<4, HALF>, X, Y, signs, n_blocks, N, scale);
    case 256: return cudaLaunchKernelEx(&cfg, hadamard_kernel<8, HALF>, X, Y, signs, n_blocks, N, scale);
    case 512: return cudaLaunchKernelEx(&cfg, hadamard_kernel<16, HALF>, X, Y, signs, n_blocks, N, scale);
    default: return cudaLaunchKernelEx(&cfg, hadamard_kernel<32, HALF>, X, Y, signs, n_blocks, N, scale);
  }
}

}  // namespace

sbvr_status launch_hadamard(const void* X, void* Y, int dtype, int rows, int N, int b, const int8_t* signs,
                            cudaStream_t st) {
  const long n_blocks = (long)rows * (N / b);
  if (n_blocks == 0) return SBVR_OK;
  cudaError_t e = dtype == SBVR_F16 ? launch_h<true>(b, X, Y, signs, n_blocks, N, st)
                                    : launch_h<false>(b, X, Y, signs, n_blocks, N, st);
  if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "hadamard launch: %s", cudaGetErrorString(e));
  return check_launch("hadamard_kernel");
}

}  // namespace sbvr
