// Step-0 microbenchmarks: which instruction pipe bounds an
// SBVR GEMV formulation on sm_100a.  Each test runs one full wave (148 SMs x
// `occ` CTAs) and reports lane-ops per SM-clock measured with clock64() inside
// the kernel, plus a streaming read bandwidth test timed with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step0 step0.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// kind: 0 LOP3, 1 POPC, 2 IMAD, 3 I2F, 4 IMMA m16n8k32 u8, 5 DFMA, 6 SHFL, 7 HMMA m16n8k16
__global__ void pipe_test(int kind, uint32_t seed, uint32_t* out, long long* cyc) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  uint32_t b = seed ^ 0x1234567u, c = seed + 77u;
  __syncthreads();
  long long t0 = clock64();
  if (kind == 0) {
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = lop3(a[i], b, c);
    }
  } else if (kind == 1) {
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = __popc(a[i] ^ b) + a[i];
    }
  } else if (kind == 2) {
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = a[i] * b + c;
    }
  } else if (kind == 3) {
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = 0.f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) { f[i] += __int2float_rn((int)(a[i] + it)); }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __float_as_uint(f[i]);
  } else if (kind == 4) {
    int d[4][4];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int i = 0; i < 4; ++i) d[m][i] = 0;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+r"(d[m][0]), "+r"(d[m][1]), "+r"(d[m][2]), "+r"(d[m][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4 + (m & 1)]), "r"(a[6]));
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = d[m][0] + d[m][1] + d[m][2] + d[m][3];
  } else if (kind == 5) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (double)a[i];
    double y = (double)b * 1e-9, z = (double)c;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, z);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (uint32_t)(long long)x[i];
  } else if (kind == 6) {
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 3));
    }
  } else if (kind == 7) {
    float d[4][4];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int i = 0; i < 4; ++i) d[m][i] = 0.f;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[m][0]), "+f"(d[m][1]), "+f"(d[m][2]), "+f"(d[m][3])
            : "r"(a[0] & 0x3c003c00u), "r"(a[1] & 0x3c003c00u), "r"(a[2] & 0x3c003c00u), "r"(a[3] & 0x3c003c00u),
              "r"(a[4 + (m & 1)] & 0x3c003c00u), "r"(a[6] & 0x3c003c00u));
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = __float_as_uint(d[m][0] + d[m][1] + d[m][2] + d[m][3]);
  }
  long long t1 = clock64();
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r ^= a[i];
  if (r == 0xdeadbeefu) out[blockIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void read_bw(const int4* __restrict__ p, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { int4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int l2 = 0, clk = 0, memclk = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d, \"memclock_khz\": %d, \"smem_optin\": %zu}\n",
         prop.name, prop.multiProcessorCount, l2, clk, memclk, prop.sharedMemPerBlockOptin);
  const int sms = prop.multiProcessorCount;
  uint32_t* out; long long* cyc;
  CK(cudaMalloc(&out, 1 << 20)); CK(cudaMalloc(&cyc, 1 << 20));
  const char* names[] = {"LOP3", "POPC", "IMAD", "I2F", "IMMA16832_u8", "DFMA", "SHFL", "HMMA16816_f16"};
  // ops per thread per kernel (lane-ops for ALU kinds; warp-MMA count*32 for MMA kinds)
  const double ops_per_thread[] = {8.0 * ITERS, 8.0 * ITERS, 8.0 * ITERS, 8.0 * ITERS, 4.0 * (ITERS / 4),
                                   8.0 * (ITERS / 4), 8.0 * (ITERS / 4), 4.0 * (ITERS / 4)};
  for (int kind = 0; kind < 8; ++kind) {
    for (int occ : {4, 8}) {
      int threads = 256, blocks = sms * occ;
      pipe_test<<<blocks, threads>>>(kind, 12345u, out, cyc);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      pipe_test<<<blocks, threads>>>(kind, 12345u, out, cyc);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long* h = new long long[blocks];
      cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
      long long mx = 0; double avg = 0;
      for (int i = 0; i < blocks; ++i) { if (h[i] > mx) mx = h[i]; avg += h[i]; }
      avg /= blocks;
      delete[] h;
      double warp_ops = ops_per_thread[kind] * threads / 32.0 * occ;  // warp-instr per SM
      double per_clk = warp_ops / (double)mx;
      double lane_per_clk = per_clk * 32.0;
      double ghz = (double)mx / (ms * 1e6);  // approx SM clock (single wave)
      printf("{\"test\": \"%s\", \"occ_ctas\": %d, \"warp_instr_per_sm_clk\": %.3f, \"lane_ops_per_sm_clk\": %.1f, "
             "\"cycles_max\": %lld, \"cycles_avg\": %.0f, \"ms\": %.4f, \"est_ghz\": %.3f}\n",
             names[kind], occ, per_clk, lane_per_clk, mx, avg, ms, ghz);
    }
  }
  // streaming read bandwidth
  size_t bytes = (size_t)4 << 30;
  int4* buf; CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  size_t n16 = bytes / 16;
  for (int occ : {4, 8, 16}) {
    for (int threads : {256, 512}) {
      int blocks = sms * occ * 256 / threads;
      read_bw<<<blocks, threads>>>(buf, n16, out);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        read_bw<<<blocks, threads>>>(buf, n16, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("{\"test\": \"read_bw_ldg128\", \"blocks\": %d, \"threads\": %d, \"GBps\": %.1f}\n", blocks, threads,
             bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
