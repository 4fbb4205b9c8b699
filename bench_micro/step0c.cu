// Step-0c: IMMA.16832 latency and throughput with the SBVR operand shape (A from LOP3 masks of
// words held in registers, B fixed), varying independent accumulator chains per warp and warps/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void k(uint32_t seed, uint32_t* out, long long* cyc, int iters) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = seed * (threadIdx.x + 7 * i + 1) ^ (0x9E3779B9u * i);
  const uint32_t b0 = seed ^ 0x80808080u, b1 = seed ^ 0x40404040u;
  int d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint32_t m0 = 0x01010101u << (2 * s), m1 = 0x01010101u << (2 * s + 1);
        const uint32_t x0 = w[(2 * c) & 7], x1 = w[(2 * c + 1) & 7];
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
            : "r"(x0 & m0), "r"(x1 & m0), "r"(x0 & m1), "r"(x1 & m1), "r"(b0), "r"(b1));
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = __funnelshift_l(w[i], w[i], 1);  // new words each iteration
  }
  long long t1 = clock64();
  int r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r += d[c][0] ^ d[c][1] ^ d[c][2] ^ d[c][3];
  if (r == 0x7fffffff) out[blockIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps_per_sm, uint32_t* out, long long* cyc) {
  const int iters = 512;
  int blocks = 148, threads = 32 * warps_per_sm;
  k<CH><<<blocks, threads>>>(1234u, out, cyc, iters);
  cudaDeviceSynchronize();
  k<CH><<<blocks, threads>>>(1234u, out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double mma = (double)iters * 4 * CH * warps_per_sm;
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"imma_per_sm_clk\": %.3f, \"cycles_per_mma_per_warp\": %.1f, \"err\": \"%s\"}\n",
         CH, warps_per_sm, mma / avg, avg / (iters * 4 * CH), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 20);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
  }
  return 0;
}
