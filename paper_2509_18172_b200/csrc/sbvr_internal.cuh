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
// One packed buffer of "units".  A unit is (band b of up to 4 row tiles of 16 rows, group g):
//   [nb tiles x 256*K bytes of planes][nb x 64 B scale/bias][nb x 16 B ratio index]
// Full bands come first (unit index b*NG + g, all the same size), then the tail band (M % 64).
struct Layout {
  int M, N, K, MT, NG, n_full, tail_nb, n_bands;
  __host__ __device__ Layout(int M_, int N_, int K_) : M(M_), N(N_), K(K_) {
    MT = M / kTileRows;
    NG = N / kG;
    n_full = MT / kBandTiles;
    tail_nb = MT % kBandTiles;
    n_bands = n_full + (tail_nb ? 1 : 0);
  }
  __host__ __device__ long unit_bytes(int nb) const { return (long)nb * (256L * K + 80); }
  __host__ __device__ long unit_off(int b, int g) const {
    if (b < n_full) return ((long)b * NG + g) * unit_bytes(kBandTiles);
    return (long)n_full * NG * unit_bytes(kBandTiles) + (long)g * unit_bytes(tail_nb);
  }
  __host__ __device__ long total_bytes() const {
    return (long)n_full * NG * unit_bytes(kBandTiles) + (tail_nb ? (long)NG * unit_bytes(tail_nb) : 0L);
  }
  __host__ __device__ int band_tiles(int b) const { return b < n_full ? kBandTiles : tail_nb; }
  // byte offset of the 32-bit word holding plane t, word c (elements 32c..32c+31) of (row, group)
  __host__ __device__ long plane_byte(int row, int g, int t, int c) const {
    const int rt = row / kTileRows, b = rt / kBandTiles, i = rt % kBandTiles, r16 = row % kTileRows;
    const int lane = 4 * (r16 % 8) + c, h = r16 / 8, q = t / 2;
    const bool last_odd = (K & 1) && (q == K / 2);
    const long base = unit_off(b, g) + (long)i * 256 * K + (long)q * 512;
    return last_odd ? base + lane * 8 + h * 4 : base + lane * 16 + ((t % 2) * 2 + h) * 4;
  }
  __host__ __device__ long sb_byte(int row, int g) const {
    const int rt = row / kTileRows, b = rt / kBandTiles, i = rt % kBandTiles, r16 = row % kTileRows;
    return unit_off(b, g) + (long)band_tiles(b) * 256 * K + i * 64 + (2 * (r16 % 8) + r16 / 8) * 4;
  }
  __host__ __device__ long ri_byte(int row, int g) const {
    const int rt = row / kTileRows, b = rt / kBandTiles, i = rt % kBandTiles, r16 = row % kTileRows;
    return unit_off(b, g) + (long)band_tiles(b) * (256L * K + 64) + i * 16 + 2 * (r16 % 8) + r16 / 8;
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
