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
constexpr int kBandTiles = 4;    // tiles per band (B-operand reuse across 64 rows)
constexpr int kMaxK = 8;
constexpr int kMaxT = 16;

// ------------------------------------------------------------------ device weight layout (sbvr.h)
struct Layout {
  int M, N, K, MT, NG, n_bands;
  __host__ __device__ Layout(int M_, int N_, int K_) : M(M_), N(N_), K(K_) {
    MT = M / kTileRows;
    NG = N / kG;
    n_bands = (MT + kBandTiles - 1) / kBandTiles;
  }
  __host__ __device__ int band_tiles(int b) const {
    int r = MT - kBandTiles * b;
    return r < kBandTiles ? r : kBandTiles;
  }
  // linear tile index of (row tile rt, group g)
  __host__ __device__ long tile(int rt, int g) const {
    int b = rt / kBandTiles;
    return (long)kBandTiles * b * NG + (long)g * band_tiles(b) + (rt - kBandTiles * b);
  }
  __host__ __device__ long tiles() const { return (long)MT * NG; }
  __host__ __device__ long tile_words() const { return 64L * K; }
  // word offset (within the planes array) of plane t, word c of (row, group)
  __host__ __device__ long plane_word(int row, int g, int t, int c) const {
    long L = tile(row / kTileRows, g);
    int r16 = row % kTileRows;
    int lane = 4 * (r16 % 8) + c;
    int h = r16 / 8;
    int q = t / 2;
    int last_odd = (K & 1) && (q == K / 2);
    long base = L * tile_words() + (long)q * 128;  // 32 lanes x 4 words per full chunk
    if (last_odd) return base + lane * 2 + h;
    return base + lane * 4 + (t % 2) * 2 + h;
  }
  // index into scale_bias / ratio_idx
  __host__ __device__ long meta(int row, int g) const {
    long L = tile(row / kTileRows, g);
    int r16 = row % kTileRows;
    return 16 * L + 2 * (r16 % 8) + r16 / 8;
  }
};

// ------------------------------------------------------------------ error plumbing
sbvr_status set_error(sbvr_status s, const char* fmt, ...);
sbvr_status check_launch(const char* what);

// ------------------------------------------------------------------ kernel launchers (one per .cu)
sbvr_status launch_encode_vector(const uint16_t* x, int T, int N, int l, uint32_t* planes, float* scales,
                                 cudaStream_t st);
sbvr_status launch_encode_weights(const sbvr_encode_config* cfg, const void* W, int dtype, int M, int N,
                                  const sbvr_weights* out, double* group_mse, cudaStream_t st);
sbvr_status launch_ratio_table(float* ratio_pow, int n_ratio, int K, cudaStream_t st);
sbvr_status launch_gemv_popc(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, int32_t* P_debug,
                             cudaStream_t st);
sbvr_status launch_gemv_fp16x(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, cudaStream_t st);
sbvr_status launch_gemv_imma(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                             int32_t* P_debug, cudaStream_t st);
size_t imma_workspace_bytes(const sbvr_weights* w, int T);

}  // namespace sbvr
