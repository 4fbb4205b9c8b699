// tc_probe.cu -- validates the tcgen05 building blocks the SBVR tensor-memory GEMV relies on:
//   A [128 x 32] u8 written to TMEM with tcgen05.st.32x32b (thread = row), B [32 x 8] u8 in shared
//   memory (K-major canonical, no swizzle), tcgen05.mma.cta_group::1.kind::i8 M=128 N=8 K=32,
//   commit -> mbarrier, tcgen05.ld of D [128 x 8] s32.  Compares with a CPU reference.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint32_t* __restrict__ A, const uint8_t* __restrict__ B, int32_t* __restrict__ D,
                      int lbo, int sbo, int accumulate_twice) {
  __shared__ __align__(1024) uint8_t sB[1024];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B^T [n=8][k=32] K-major canonical: core matrix = 8 rows x 16 B; k-chunk j at j*lbo
  for (int i = tid; i < 8 * 32; i += blockDim.x) {
    const int n = i / 32, k = i % 32;
    sB[(k / 16) * lbo + n * 16 + (k % 16)] = B[k * 8 + n];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // sB written by generic proxy, read by MMA
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = s_tmem;
  const uint32_t tA = tbase, tD = tbase + 32;
  // A row `tid`: 8 u32 columns, k = 4*col + byte
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = A[tid * 8 + i];
  const uint32_t taddr = tA + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(a[0]),
               "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t sa = smem_u32(sB);
    uint64_t desc = 0;
    desc |= (uint64_t)((sa >> 4) & 0x3fff);
    desc |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    desc |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    desc |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
    const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | (1u << 17) | (8u << 24);  // S32 acc, u8 x u8, N=8, M=128
    for (int rep = 0; rep < (accumulate_twice ? 2 : 1); ++rep) {
      const uint32_t en = rep;  // first: overwrite, second: accumulate
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
          "r"(tA), "l"(desc), "r"(idesc), "r"(en));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&s_bar))
                 : "memory");
  }
  // wait for the MMA
  asm volatile(
      "{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT;\n}\n" ::"r"(
          smem_u32(&s_bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t d[8];
  const uint32_t tdaddr = tD + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
               : "r"(tdaddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < 8; ++n) D[tid * 8 + n] = (int32_t)d[n];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(64));
}

int main() {
  uint32_t hA[128 * 8];
  uint8_t hB[32 * 8];
  srand(1);
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (uint32_t)rand() * 2654435761u;
  for (int i = 0; i < 256; ++i) hB[i] = (uint8_t)(rand() & 0xff);
  int64_t ref[128][8];
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < 8; ++n) {
      int64_t s = 0;
      for (int k = 0; k < 32; ++k) {
        const uint32_t w = hA[r * 8 + k / 4];
        const int av = (w >> (8 * (k % 4))) & 0xff;
        s += (int64_t)av * hB[k * 8 + n];
      }
      ref[r][n] = s;
    }
  uint32_t* dA; uint8_t* dB; int32_t* dD;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, 128 * 8 * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  int cfgs[][3] = {{128, 256, 0}, {256, 128, 0}, {128, 256, 1}};
  for (auto& c : cfgs) {
    cudaMemset(dD, 0, 128 * 8 * 4);
    probe<<<1, 128>>>(dA, dB, dD, c[0], c[1], c[2]);
    cudaError_t e = cudaDeviceSynchronize();
    int32_t hD[128 * 8];
    cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < 8; ++n)
        if (hD[r * 8 + n] != (int32_t)(ref[r][n] * (c[2] ? 2 : 1))) ++bad;
    printf("{\"lbo\": %d, \"sbo\": %d, \"accum2\": %d, \"err\": \"%s\", \"mismatches\": %d, \"d00\": %d, \"ref00\": %lld}\n",
           c[0], c[1], c[2], cudaGetErrorString(e), bad, hD[0], (long long)ref[0][0]);
  }
  return 0;
}
