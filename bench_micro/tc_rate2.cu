// tc_rate2.cu -- what paces small-N tcgen05.mma on sm_100a?  Round 1 (tc_rate.cu) measured a flat
// ~46 cycles per M=128 K=32 kind::i8 MMA for every N <= 64 with 4 accumulators.  This sweep separates
// the candidates: independent accumulator chains (1..16), N (8..256), A from TMEM (TS) or SMEM (SS),
// kind::i8 vs kind::f16, and M = 64 vs 128.  One thread per CTA issues `iters` x 16 MMAs round-robin over
// `chains` accumulators, one commit at the end; cycles = first issue -> commit's mbarrier completion.
// Every SM runs the same CTA (grid 148).  Output: one JSON line per configuration.
#include <cstdint>
#include <cstdio>
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

// KIND 0 = i8 (s32 += u8*u8), 1 = f16 (f32 += f16*f16)
template <int KIND, bool TS>
__global__ void rate(int M, int N, int chains, int iters, long long* out, int ncols) {
  extern __shared__ __align__(1024) uint8_t sm[];   // A: 128 x 32 B (4 KB), B: up to 256 x 32 B (8 KB)
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4096 + 8192; i += blockDim.x) sm[i] = KIND ? 0 : (uint8_t)(i * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(ncols));
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
  // instruction descriptor: D fmt (bits 4-5: 1 = f32, 2 = s32), A/B fmt (7-9, 10-12: f16 = 0, u8 = 0),
  // N>>3 at 17, M>>4 at 24
  const uint32_t idesc = (KIND ? (1u << 4) : (2u << 4)) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint32_t sA = smem_u32(sm), sB = smem_u32(sm + 4096);
  const uint64_t bd = desc(sB, 128, 256);
  const uint64_t ad = desc(sA, 128, 256);
  // D regions: chains x N columns from column 128 (A in TMEM uses columns 0..127)
  if (tid == 0) {
    long long t0 = clock64();
    int ch = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const uint32_t tD = tm + 32 + ch * N;
        const uint32_t en = it > 0 || m >= chains ? 1u : 0u;
        if (TS) {
          if (KIND == 0)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(tD), "r"(tm + 8 * (m & 3)), "l"(bd), "r"(idesc), "r"(en) : "memory");
          else
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(tD), "r"(tm + 8 * (m & 3)), "l"(bd), "r"(idesc), "r"(en) : "memory");
        } else {
          if (KIND == 0)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tD), "l"(ad), "l"(bd), "r"(idesc), "r"(en) : "memory");
          else
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tD), "l"(ad), "l"(bd), "r"(idesc), "r"(en) : "memory");
        }
        ch = ch + 1 == chains ? 0 : ch + 1;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(ncols));
}

template <int KIND, bool TS>
static void run(int M, int N, int chains, int per_sm = 1) {
  static long long* d = nullptr;
  if (!d) cudaMalloc(&d, 4 * 148 * sizeof(long long));
  long long h[4 * 148];
  const int ncols = 512 / per_sm;
  if (32 + chains * N > ncols) return;
  const int iters = 128;
  auto k = rate<KIND, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<148 * per_sm, 128, 16384>>>(M, N, chains, iters, d, ncols);
  k<<<148 * per_sm, 128, 16384>>>(M, N, chains, iters, d, ncols);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(long long) * 148 * per_sm, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148 * per_sm; ++i) avg += h[i];
  avg /= 148 * per_sm;
  printf("{\"kind\": \"%s\", \"A\": \"%s\", \"M\": %d, \"N\": %d, \"chains\": %d, \"ctas_per_sm\": %d, "
         "\"cycles_per_mma_per_cta\": %.2f, \"sm_cycles_per_mma\": %.2f, \"floor_guide\": %.1f, \"err\": \"%s\"}\n",
         KIND ? "f16" : "i8", TS ? "tmem" : "smem", M, N, chains, per_sm, avg / (iters * 16.0),
         avg / (iters * 16.0) / per_sm, (M > 128 ? M : 128) * N / 256.0, cudaGetErrorString(e));
  fflush(stdout);
}


// TMEM load / store throughput: `nw` warps (lane quarter = warp % 4), each repeatedly moves `cols`
// 32-bit columns of its 32 lanes (tcgen05.ld/st 32x32b.x32 = 32 columns per instruction), 128 bytes per
// lane per instruction.  Bytes per SM-cycle = nw * 32 * cols * 4 * iters / cycles.
template <bool LD>
__global__ void tmem_bw(int iters, long long* out, unsigned int* sink) {
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = tid * i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (LD) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                       "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
                       "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                       "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
                     : "r"(tm + 32 * c) : "memory");
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + 32 * c),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                     "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                     "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                     "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                     : "memory");
      }
    }
    if (LD) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    else asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  unsigned int acc = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) acc += v[i];
  if (acc == 0x12345678u) sink[0] = acc;
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
}

template <bool LD>
static void run_bw(int nw) {
  static long long* d = nullptr;
  static unsigned int* sk = nullptr;
  if (!d) { cudaMalloc(&d, 148 * sizeof(long long)); cudaMalloc(&sk, 4); }
  long long h[148];
  const int iters = 256;
  tmem_bw<LD><<<148, nw * 32>>>(iters, d, sk);
  tmem_bw<LD><<<148, nw * 32>>>(iters, d, sk);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double bytes = (double)nw * 32 * 128 * 4 * iters;
  printf("{\"test\": \"tmem_%s\", \"warps\": %d, \"bytes_per_sm_cycle\": %.1f, \"err\": \"%s\"}\n", LD ? "ld" : "st", nw,
         bytes / avg, cudaGetErrorString(e));
  fflush(stdout);
}


// one CTA per SM, `nis` issuing warps (lane 0 of warps 0..nis-1), each round-robin over 2 accumulators of
// its own; A in TMEM (columns 0..31), D from column 32 + warp * 2N
__global__ void rate_multi(int N, int nis, int iters, long long* out) {
  __shared__ __align__(1024) uint8_t sm[8192];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 8) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[tid])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  const uint64_t bd = desc(smem_u32(sm), 128, 256);
  if (lane == 0 && warp < nis) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const uint32_t tD = tm + 32 + (warp * 2 + (m & 1)) * N;
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tD), "r"(tm + 8 * (m & 3)), "l"(bd), "r"(idesc), "r"(1u) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])) : "memory");
    mbar_wait(&bar[warp], 0);
    long long t1 = clock64();
    if (warp == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

static void run_multi(int N, int nis) {
  static long long* d = nullptr;
  if (!d) cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  if (32 + nis * 2 * N > 512) return;
  const int iters = 128;
  rate_multi<<<148, 256>>>(N, nis, iters, d);
  rate_multi<<<148, 256>>>(N, nis, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("{\"test\": \"multi_issuer_one_cta\", \"N\": %d, \"issuers\": %d, \"sm_cycles_per_mma\": %.2f, \"err\": \"%s\"}\n",
         N, nis, avg / (iters * 16.0) / nis, cudaGetErrorString(e));
  fflush(stdout);
}

int main() {
  for (int N : {16, 32, 64}) for (int nis : {1, 2, 4, 8}) run_multi(N, nis);
  return 0;
  for (int per_sm : {1, 2, 4})
    for (int N : {16, 32, 64}) {
      run<0, true>(128, N, 2, per_sm);
      run<0, false>(128, N, 2, per_sm);
    }
  run<0, true>(128, 128, 1, 2);
  run<0, true>(128, 256, 1, 1);
  return 0;
}
