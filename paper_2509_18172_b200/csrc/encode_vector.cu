// encode_vector.cu -- online activation conversion, §4.3, Eq. 12.
//
// One warp per activation group of 128 elements.  Lane L holds elements L, 32+L, 64+L, 96+L,
// so one __ballot_sync per (plane j, word c) produces word c of bit-plane j directly:
//   absmax (warp max-reduce, exact) -> s_x = absmax / (2^(l-1)-1)  (IEEE fp32 divide, reading A10)
//   z = clamp(rne(x / s_x))  (cvt.rni, reading A12) -> planes = l-bit two's complement of z
// Output: planes [T][N/G][l][4] (lane 4j+c stores word (j, c): one coalesced 128-byte store),
// scales [T][N/G].  Memory-bound: 2N bytes in, (l/8 + 4/G) N bytes out.
#include "sbvr_internal.cuh"

namespace sbvr {

#ifndef SBVR_ENCVEC_THREADS
#define SBVR_ENCVEC_THREADS 32
#endif
// One warp per CTA by default: a CTA this small (~1K registers) fits beside a persistent GEMV CTA that leaves a few
// registers of the SM free (sbvr_gemv_group), so the conversion never holds an SM that the GEMV of the next step
// needs (256-thread CTAs took a whole SM from the grouped GEMV: its CTAs there started ~8 us late).
__global__ void __launch_bounds__(SBVR_ENCVEC_THREADS) encode_vector_kernel(const uint16_t* __restrict__ x, int total_groups, int l,
                                                            uint32_t* __restrict__ planes,
                                                            float* __restrict__ scales) {
  // programmatic dependent launch: let the next kernel (the GEMV that reads our planes) be scheduled at once -- its
  // CTAs take SMs as the previous GEMV's CTAs retire and start streaming their weights, which do not depend on us;
  // its griddepcontrol.wait still waits for this grid to complete.  We wait for the previous kernel before writing:
  // it may still be reading the planes we overwrite.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // group index over [T][N/G]
  if (q >= total_groups) return;
  const uint16_t* xg = x + (size_t)q * kG;                      // groups are contiguous in [T][N]
  float v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = __half2float(__ushort_as_half(__ldg(xg + 32 * c + lane)));
  float a = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
  const int zmax = (1 << (l - 1)) - 1;
  const float sx = (a != 0.0f) ? __fdiv_rn(a, (float)zmax) : 0.0f;
  const uint32_t lmask = (1u << l) - 1u;
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
  if (lane < 4 * l) planes[(size_t)q * 4 * l + lane] = mine;
  if (lane == 0) scales[q] = sx;
}

sbvr_status launch_encode_vector(const uint16_t* x, int T, int N, int l, uint32_t* planes, float* scales,
                                 cudaStream_t st) {
  const int groups = T * (N / kG);
  const int blocks = (groups * 32 + SBVR_ENCVEC_THREADS - 1) / SBVR_ENCVEC_THREADS;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(SBVR_ENCVEC_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, encode_vector_kernel, x, groups, l, planes, scales);
  if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "encode_vector launch: %s", cudaGetErrorString(e));
  return check_launch("encode_vector_kernel");
}

}  // namespace sbvr
