// Internal declarations shared by the libsbvr translation units (never by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstddef>

#include "../../include/sbvr.h"

namespace sbvr {

constexpr int kG = 128;          // group size supported by the kernels
constexpr int kWPG = kG / 32;    // 32-bit words per plane per group
constexpr int kTileRows = 16;    // rows per tile (mma m16)
constexpr int kMaxK = 8;
constexpr int kMaxT = 256;      // tokens per batched call (prefill chunks); kernels loop over passes

// ------------------------------------------------------------------ device weight layout (sbvr.h)
// One packed buffer of "units".  A unit is (row block rb of up to 128 rows, group g) stored as
//   [R rows x 16K bytes: row r's K plane chunks (16 B = 4 words each), chunk t at t ^ swz(r)]
//   [R x 4 B scale/bias][R x 1 B ratio index]
// with R = 128 for full blocks; the last block holds M % 128 rows (a multiple of 16).  Units are
// ordered rb-major (unit index rb*NG + g), so a row block's groups are consecutive.
constexpr int kRowBlock = 128;

__host__ __device__ __forceinline__ int chunk_swizzle(int K, int r) {
  // makes the 16-byte chunk loads of 8 consecutive rows hit 8 distinct bank groups
  return K == 2 ? ((r >> 2) & 1) : K == 4 ? ((r >> 1) & 3) : K == 6 ? ((r >> 2) & 1) : K == 8 ? (r & 7) : 0;
}

struct Layout {
  int M, N, K, NG, n_rb, n_full, tail_rows;
  __host__ __device__ Layout(int M_, int N_, int K_) : M(M_), N(N_), K(K_) {
    NG = N / kG;
    n_full = M / kRowBlock;
    tail_rows = M % kRowBlock;
    n_rb = n_full + (tail_rows ? 1 : 0);
  }
  __host__ __device__ int rows_in(int rb) const { return rb < n_full ? kRowBlock : tail_rows; }
  __host__ __device__ long unit_bytes(int rows) const { return (long)rows * (16L * K + 5); }
  __host__ __device__ long unit_off(int rb, int g) const {
    if (rb < n_full) return ((long)rb * NG + g) * unit_bytes(kRowBlock);
    return (long)n_full * NG * unit_bytes(kRowBlock) + (long)g * unit_bytes(tail_rows);
  }
  __host__ __device__ long total_bytes() const {
    return (long)n_full * NG * unit_bytes(kRowBlock) + (tail_rows ? (long)NG * unit_bytes(tail_rows) : 0L);
  }
  // byte offset of the 32-bit word holding plane t, word c (elements 32c..32c+31) of (row, group)
  __host__ __device__ long plane_byte(int row, int g, int t, int c) const {
    const int rb = row / kRowBlock, r = row % kRowBlock;
    return unit_off(rb, g) + (long)r * 16 * K + 16 * (t ^ chunk_swizzle(K, r)) + 4 * c;
  }
  __host__ __device__ long sb_byte(int row, int g) const {
    const int rb = row / kRowBlock, r = row % kRowBlock;
    return unit_off(rb, g) + (long)rows_in(rb) * 16 * K + 4 * r;
  }
  __host__ __device__ long ri_byte(int row, int g) const {
    const int rb = row / kRowBlock, r = row % kRowBlock;
    return unit_off(rb, g) + (long)rows_in(rb) * (16L * K + 4) + r;
  }
};

// SBVR_META_INDEXED records: [R x 16K planes][R x 1 B coefficient-table index]
struct IdxLayout {
  int M, N, K, NG, n_full, tail_rows;
  __host__ __device__ IdxLayout(int M_, int N_, int K_) : M(M_), N(N_), K(K_) {
    NG = N / kG;
    n_full = M / kRowBlock;
    tail_rows = M % kRowBlock;
  }
  __host__ __device__ int rows_in(int rb) const { return rb < n_full ? kRowBlock : tail_rows; }
  __host__ __device__ long unit_bytes(int rows) const { return (long)rows * (16L * K + 1); }
  __host__ __device__ long unit_off(int rb, int g) const {
    if (rb < n_full) return ((long)rb * NG + g) * unit_bytes(kRowBlock);
    return (long)n_full * NG * unit_bytes(kRowBlock) + (long)g * unit_bytes(tail_rows);
  }
  __host__ __device__ long total_bytes() const {
    return (long)n_full * NG * unit_bytes(kRowBlock) + (tail_rows ? (long)NG * unit_bytes(tail_rows) : 0L);
  }
  __host__ __device__ long plane_byte(int row, int g, int t, int c) const {
    const int rb = row / kRowBlock, r = row % kRowBlock;
    return unit_off(rb, g) + (long)r * 16 * K + 16 * (t ^ chunk_swizzle(K, r)) + 4 * c;
  }
  __host__ __device__ long idx_byte(int row, int g) const {
    const int rb = row / kRowBlock, r = row % kRowBlock;
    return unit_off(rb, g) + (long)rows_in(rb) * 16 * K + r;
  }
};
constexpr int kMaxTable = 256;
constexpr size_t kTableBytes = (1 + 2 * kMaxTable) * 4;

// ------------------------------------------------------------------ error plumbing
sbvr_status set_error(sbvr_status s, const char* fmt, ...);
sbvr_status check_launch(const char* what);

// ------------------------------------------------------------------ kernel launchers (one per .cu)
sbvr_status launch_encode_vector(const uint16_t* x, int T, int N, int l, uint32_t* planes, float* scales,
                                 cudaStream_t st);
sbvr_status launch_encode_weights(const sbvr_encode_config* cfg, const void* W, int dtype, int M, int N,
                                  const sbvr_weights* out, double* group_mse, int cache_size, double cache_alpha,
                                  uint8_t* group_hit, cudaStream_t st);
sbvr_status launch_ratio_table(float* ratio_pow, int n_ratio, int K, cudaStream_t st);
sbvr_status launch_encode_indexed(const sbvr_encode_config* cfg, int n_table, const void* W, int dtype, int M, int N,
                                  const sbvr_weights* out, double* group_mse, uint32_t* cand, cudaStream_t st);
sbvr_status launch_gemv_popc(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, int32_t* P_debug,
                             cudaStream_t st);
sbvr_status launch_gemv_fp16x(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, cudaStream_t st);
sbvr_status launch_gemv_tc(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                           int32_t* P_debug, cudaStream_t st);
size_t tc_workspace_bytes(const sbvr_weights* w, int T);
// fused row-shard all-gather epilogue: every y value also lands in each rank's full-y buffer (dist.py)
struct PeerOut {
  float* y[8];          // device pointers (symmetric memory; own rank included), each [T][M_full] fp32
  int n, row_offset, M_full;
};
sbvr_status launch_gemv_mma(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                            int32_t* P_debug, cudaStream_t st, const PeerOut* peers = nullptr,
                            const sbvr_weights* next_w = nullptr);
size_t mma_workspace_bytes(const sbvr_weights* w, int T);
sbvr_status launch_gemv_pipe(const sbvr_weights* w, const sbvr_act* x, float* y, void* ws, int32_t* P_debug,
                             cudaStream_t st);
size_t pipe_workspace_bytes(const sbvr_weights* w);
bool pipe_supported(const sbvr_weights* w, const sbvr_act* x);
sbvr_status launch_gemv_zt(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                           int32_t* T_debug, cudaStream_t st);
size_t zt_workspace_bytes(const sbvr_weights* w, int T);
bool zt_supported(const sbvr_weights* w, const sbvr_act* x);
struct GroupPeers {       // fused all-gather of a grouped GEMV: y[i * n + j] = rank j's full y of problem i
  float* const* y;
  int n;
  const int32_t* row_offset;   // [problem] this rank's first row in the full y
};
sbvr_status launch_gemv_group(const sbvr_gemv_problem* pr, int n, void* ws, size_t ws_bytes, cudaStream_t st,
                              const GroupPeers* peers = nullptr);
size_t group_workspace_bytes(const sbvr_gemv_problem* pr, int n);
sbvr_status launch_prefill(const sbvr_weights* w, const uint16_t* X, int T, float* Y, void* ws, size_t ws_bytes,
                           cudaStream_t st);
size_t prefill_workspace_bytes(const sbvr_weights* w, int T);
sbvr_status launch_hadamard(const void* X, void* Y, int dtype, int rows, int N, int b, const int8_t* signs,
                            cudaStream_t st);

}  // namespace sbvr
