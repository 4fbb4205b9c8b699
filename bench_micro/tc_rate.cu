// tc_rate.cu -- throughput and latency of tcgen05.mma.cta_group::1.kind::i8 M=128 K=32 for
// several N, with A in tensor memory (TS) or shared memory (SS), on every SM at once.
//   throughput: one thread issues `iters` x 16 MMAs (4 independent accumulators), one commit at
//               the end; cycles from first issue to the commit's mbarrier completion
//   latency:    one MMA, commit, wait -- repeated
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t sa, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((sa >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

template <bool TS>
__global__ void rate(int N, int iters, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];   // A: 128 x 32 B (4 KB), B: N x 32 B
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4096 + 8192; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  const uint32_t sA = smem_u32(sm), sB = smem_u32(sm + 4096);
  const uint64_t bd = desc(sB, 128, 256);
  const uint64_t ad = desc(sA, 128, 256);
  if (tid == 0) {
    uint32_t ph = 0;
    long long t0 = clock64();
    if (mode == 0) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const uint32_t tD = tm + 256 + (N <= 64 ? (m & 3) * N : (N == 128 ? (m & 1) * 128 : 0));
          const uint32_t en = (it | (m >> 2)) ? 1u : 0u;
          if (TS)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(tD), "r"(tm + 8 * (m & 3) * 4), "l"(bd), "r"(idesc), "r"(en) : "memory");
          else
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tD), "l"(ad), "l"(bd), "r"(idesc), "r"(en) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      mbar_wait(&bar, 0);
    } else {
      for (int it = 0; it < iters; ++it) {
        if (TS)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tm + 256), "r"(tm), "l"(bd), "r"(idesc), "r"(1u) : "memory");
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm + 256), "l"(ad), "l"(bd), "r"(idesc), "r"(1u) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  for (int ts = 1; ts >= 0; --ts)
    for (int N : {8, 16, 32, 64, 128, 256}) {
      for (int mode = 0; mode < 2; ++mode) {
        const int iters = mode == 0 ? 256 : 64;
        auto k = ts ? rate<true> : rate<false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
        k<<<148, 128, 16384>>>(N, iters, mode, d);
        k<<<148, 128, 16384>>>(N, iters, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double per = mode == 0 ? avg / (iters * 16.0) : avg / iters;
        printf("{\"A\": \"%s\", \"N\": %d, \"test\": \"%s\", \"cycles_per_mma\": %.2f, \"floor\": %.1f, \"err\": \"%s\"}\n",
               ts ? "tmem" : "smem", N, mode == 0 ? "throughput" : "latency(mma+commit+wait)", per, 128.0 * N / 256,
               cudaGetErrorString(e));
      }
    }
  return 0;
}
