// abi.cu -- extern "C" entry points of libsbvr (include/sbvr.h): argument validation,
// size queries, host-side layout transforms and dispatch to the kernels.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sbvr_internal.cuh"

namespace sbvr {

static thread_local char g_err[512] = "";

sbvr_status set_error(sbvr_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

sbvr_status check_launch(const char* what) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(SBVR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  return SBVR_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static sbvr_status check_weights(const sbvr_weights* w) {
  if (!w) return set_error(SBVR_ERR_INVALID_ARG, "weights descriptor is NULL");
  if (!w->data || !w->ratio_pow) return set_error(SBVR_ERR_INVALID_ARG, "weights buffer pointer is NULL");
  if (w->group_size != kG) return set_error(SBVR_ERR_UNSUPPORTED, "group_size %d (only 128)", w->group_size);
  if (w->K < 1 || w->K > kMaxK) return set_error(SBVR_ERR_UNSUPPORTED, "K=%d outside 1..8", w->K);
  if (w->n_ratio < 2 || w->n_ratio > 64 || (w->n_ratio & 1))
    return set_error(SBVR_ERR_INVALID_ARG, "n_ratio=%d must be even in 2..64", w->n_ratio);
  if (w->M <= 0 || w->N <= 0) return set_error(SBVR_ERR_SHAPE, "M=%d N=%d must be positive", w->M, w->N);
  if (w->M % kTileRows) return set_error(SBVR_ERR_SHAPE, "M=%d not a multiple of 16", w->M);
  if (w->N % kG) return set_error(SBVR_ERR_SHAPE, "N=%d not a multiple of group_size 128", w->N);
  if (!aligned16(w->data) || !aligned16(w->ratio_pow))
    return set_error(SBVR_ERR_ALIGNMENT, "weights buffers must be 16-byte aligned");
  if (w->meta_kind != SBVR_META_GROUP && w->meta_kind != SBVR_META_INDEXED)
    return set_error(SBVR_ERR_INVALID_ARG, "unknown meta_kind %d", w->meta_kind);
  if (w->meta_kind == SBVR_META_INDEXED) {
    if (!w->coef_table) return set_error(SBVR_ERR_INVALID_ARG, "indexed weights need coef_table");
    if (!aligned16(w->coef_table)) return set_error(SBVR_ERR_ALIGNMENT, "coef_table must be 16-byte aligned");
  }
  return SBVR_OK;
}

static sbvr_status check_act(const sbvr_weights* w, const sbvr_act* x, int T) {
  if (!x || !x->data) return set_error(SBVR_ERR_INVALID_ARG, "activation descriptor/data is NULL");
  if (T < 1 || T > kMaxT) return set_error(SBVR_ERR_SHAPE, "T=%d outside 1..256", T);
  if (x->N != w->N) return set_error(SBVR_ERR_SHAPE, "x.N=%d != W.N=%d", x->N, w->N);
  if (x->group_size != w->group_size)
    return set_error(SBVR_ERR_SHAPE, "x.group_size=%d != W.group_size=%d", x->group_size, w->group_size);
  if (x->kind == SBVR_ACT_SBVR) {
    if (!x->scales) return set_error(SBVR_ERR_INVALID_ARG, "SBVR activation scales are NULL");
    if (x->l < 2 || x->l > 8) return set_error(SBVR_ERR_UNSUPPORTED, "l=%d outside 2..8", x->l);
    if (!aligned16(x->data)) return set_error(SBVR_ERR_ALIGNMENT, "activation planes must be 16-byte aligned");
  } else if (x->kind == SBVR_ACT_FP16) {
    if (!aligned16(x->data)) return set_error(SBVR_ERR_ALIGNMENT, "fp16 activation must be 16-byte aligned");
  } else if (x->kind == SBVR_ACT_FP16_Q) {
    if (x->l < 2 || x->l > 8) return set_error(SBVR_ERR_UNSUPPORTED, "l=%d outside 2..8", x->l);
    if (T != 1) return set_error(SBVR_ERR_UNSUPPORTED, "in-kernel conversion (SBVR_ACT_FP16_Q) runs T = 1 (T=%d)", T);
    if (w->K < 2 || w->K > 4) return set_error(SBVR_ERR_UNSUPPORTED, "SBVR_ACT_FP16_Q: K=%d outside 2..4", w->K);
    if (!aligned16(x->data)) return set_error(SBVR_ERR_ALIGNMENT, "fp16 activation must be 16-byte aligned");
  } else {
    return set_error(SBVR_ERR_INVALID_ARG, "unknown activation kind %d", x->kind);
  }
  return SBVR_OK;
}

}  // namespace sbvr

using namespace sbvr;

extern "C" {

int32_t sbvr_abi_version(void) { return SBVR_ABI_VERSION; }

const char* sbvr_status_string(sbvr_status s) {
  switch (s) {
    case SBVR_OK: return "SBVR_OK";
    case SBVR_ERR_INVALID_ARG: return "SBVR_ERR_INVALID_ARG";
    case SBVR_ERR_SHAPE: return "SBVR_ERR_SHAPE";
    case SBVR_ERR_UNSUPPORTED: return "SBVR_ERR_UNSUPPORTED";
    case SBVR_ERR_ALIGNMENT: return "SBVR_ERR_ALIGNMENT";
    case SBVR_ERR_CUDA: return "SBVR_ERR_CUDA";
    case SBVR_ERR_WORKSPACE: return "SBVR_ERR_WORKSPACE";
  }
  return "SBVR_UNKNOWN_STATUS";
}

const char* sbvr_last_error(void) { return g_err; }

sbvr_status sbvr_weights_bytes(int32_t M, int32_t N, int32_t K, int32_t group_size, int32_t n_ratio,
                               size_t* data_bytes, size_t* ratio_pow_bytes) {
  if (!data_bytes || !ratio_pow_bytes)
    return set_error(SBVR_ERR_INVALID_ARG, "output pointer is NULL");
  if (group_size != kG) return set_error(SBVR_ERR_UNSUPPORTED, "group_size %d (only 128)", group_size);
  if (K < 1 || K > kMaxK) return set_error(SBVR_ERR_UNSUPPORTED, "K=%d outside 1..8", K);
  if (M <= 0 || N <= 0 || M % kTileRows || N % kG)
    return set_error(SBVR_ERR_SHAPE, "M=%d must be a positive multiple of 16, N=%d of 128", M, N);
  if (n_ratio < 2 || n_ratio > 64 || (n_ratio & 1)) return set_error(SBVR_ERR_INVALID_ARG, "bad n_ratio %d", n_ratio);
  *data_bytes = (size_t)Layout(M, N, K).total_bytes();
  *ratio_pow_bytes = (size_t)n_ratio * K * 4;
  return SBVR_OK;
}

sbvr_status sbvr_weights_bytes_ex(int32_t M, int32_t N, int32_t K, int32_t group_size, int32_t n_ratio,
                                  int32_t meta_kind, size_t* data_bytes, size_t* ratio_pow_bytes, size_t* table_bytes) {
  if (!table_bytes) return set_error(SBVR_ERR_INVALID_ARG, "output pointer is NULL");
  sbvr_status s = sbvr_weights_bytes(M, N, K, group_size, n_ratio, data_bytes, ratio_pow_bytes);
  if (s != SBVR_OK) return s;
  if (meta_kind == SBVR_META_GROUP) {
    *table_bytes = 0;
  } else if (meta_kind == SBVR_META_INDEXED) {
    *data_bytes = (size_t)IdxLayout(M, N, K).total_bytes();
    *table_bytes = kTableBytes;
  } else {
    return set_error(SBVR_ERR_INVALID_ARG, "unknown meta_kind %d", meta_kind);
  }
  return SBVR_OK;
}

static sbvr_status check_encode(const sbvr_encode_config* cfg, const void* W, int32_t dtype, int32_t M, int32_t N,
                                const sbvr_weights* out) {
  if (!cfg || !W || !out) return set_error(SBVR_ERR_INVALID_ARG, "cfg/W/out is NULL");
  if (dtype != SBVR_F32 && dtype != SBVR_F16 && dtype != SBVR_BF16)
    return set_error(SBVR_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  if (cfg->K < 1 || cfg->K > 6) return set_error(SBVR_ERR_UNSUPPORTED, "encoder K=%d outside 1..6", cfg->K);
  if (cfg->group_size != kG) return set_error(SBVR_ERR_UNSUPPORTED, "group_size %d (only 128)", cfg->group_size);
  if (cfg->n_ratio < 2 || cfg->n_ratio > 64 || (cfg->n_ratio & 1))
    return set_error(SBVR_ERR_INVALID_ARG, "n_ratio=%d must be even in 2..64", cfg->n_ratio);
  if (cfg->n_scale < 1 || cfg->n_scale > 4096 || cfg->n_bias < 1 || cfg->n_bias > 4096)
    return set_error(SBVR_ERR_INVALID_ARG, "n_scale/n_bias outside 1..4096");
  if (out->M != M || out->N != N || out->K != cfg->K || out->group_size != cfg->group_size ||
      out->n_ratio != cfg->n_ratio)
    return set_error(SBVR_ERR_SHAPE, "output descriptor does not match M/N/K/group_size/n_ratio");
  return check_weights(out);
}

sbvr_status sbvr_encode_weights(const sbvr_encode_config* cfg, const void* W, int32_t dtype, int32_t M, int32_t N,
                                const sbvr_weights* out, double* group_mse, void* stream) {
  sbvr_status s = check_encode(cfg, W, dtype, M, N, out);
  if (s != SBVR_OK) return s;
  if (out->meta_kind != SBVR_META_GROUP) return set_error(SBVR_ERR_INVALID_ARG, "out must be SBVR_META_GROUP");
  return launch_encode_weights(cfg, W, dtype, M, N, out, group_mse, -1, 0.0, nullptr, (cudaStream_t)stream);   // strict or fast
}

sbvr_status sbvr_encode_weights_indexed(const sbvr_encode_config* cfg, int32_t n_table, const void* W, int32_t dtype,
                                        int32_t M, int32_t N, const sbvr_weights* out, double* group_mse,
                                        void* workspace, size_t ws_bytes, void* stream) {
  sbvr_status s = check_encode(cfg, W, dtype, M, N, out);
  if (s != SBVR_OK) return s;
  if (!cfg->strict) return set_error(SBVR_ERR_UNSUPPORTED, "the indexed encoder runs strict (fp64) only");
  if (out->meta_kind != SBVR_META_INDEXED) return set_error(SBVR_ERR_INVALID_ARG, "out must be SBVR_META_INDEXED");
  if (n_table < 1 || n_table > kMaxTable) return set_error(SBVR_ERR_INVALID_ARG, "n_table=%d outside 1..256", n_table);
  if (!workspace || ws_bytes < (size_t)8 * n_table)
    return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, (size_t)8 * n_table);
  return launch_encode_indexed(cfg, n_table, W, dtype, M, N, out, group_mse, static_cast<uint32_t*>(workspace),
                               (cudaStream_t)stream);
}

sbvr_status sbvr_encode_weights_cached(const sbvr_encode_config* cfg, int32_t cache_size, double ema_alpha,
                                       const void* W, int32_t dtype, int32_t M, int32_t N, const sbvr_weights* out,
                                       double* group_mse, uint8_t* group_hit, void* stream) {
  sbvr_status s = check_encode(cfg, W, dtype, M, N, out);
  if (s != SBVR_OK) return s;
  if (out->meta_kind != SBVR_META_GROUP) return set_error(SBVR_ERR_INVALID_ARG, "out must be SBVR_META_GROUP");
  if (!cfg->strict) return set_error(SBVR_ERR_UNSUPPORTED, "the cached encoder runs strict (fp64) only");
  if (cache_size < 0 || cache_size > 64) return set_error(SBVR_ERR_INVALID_ARG, "cache_size=%d outside 0..64", cache_size);
  if (!(ema_alpha > 0.0 && ema_alpha <= 1.0)) return set_error(SBVR_ERR_INVALID_ARG, "ema_alpha outside (0, 1]");
  return launch_encode_weights(cfg, W, dtype, M, N, out, group_mse, cache_size, ema_alpha, group_hit,
                               (cudaStream_t)stream);
}

sbvr_status sbvr_encode_vector(const uint16_t* x, int32_t T, int32_t N, int32_t group_size, int32_t l,
                               uint32_t* planes_out, float* scales_out, void* stream) {
  if (!x || !planes_out || !scales_out) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  if (group_size != kG) return set_error(SBVR_ERR_UNSUPPORTED, "group_size %d (only 128)", group_size);
  if (l < 2 || l > 8) return set_error(SBVR_ERR_UNSUPPORTED, "l=%d outside 2..8", l);
  if (T < 1 || N <= 0 || N % kG) return set_error(SBVR_ERR_SHAPE, "T=%d N=%d", T, N);
  return launch_encode_vector(x, T, N, l, planes_out, scales_out, (cudaStream_t)stream);
}

sbvr_status sbvr_gemv_workspace_bytes(const sbvr_weights* w, int32_t T, size_t* bytes) {
  if (!w || !bytes) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  if (T < 1 || T > kMaxT) return set_error(SBVR_ERR_SHAPE, "T=%d outside 1..256", T);
  if (w->M <= 0 || w->N <= 0 || w->M % kTileRows || w->N % kG)
    return set_error(SBVR_ERR_SHAPE, "bad M/N %d/%d", w->M, w->N);
  const size_t a = tc_workspace_bytes(w, T), b = mma_workspace_bytes(w, T), c = pipe_workspace_bytes(w);
  *bytes = a > b ? a : b;
  if (c > *bytes) *bytes = c;
  if (w->K <= 4) {
    const size_t d = zt_workspace_bytes(w, T);
    if (d > *bytes) *bytes = d;
  }
  if (w->M % kRowBlock == 0) {           // the grouped kernel serves large batch-1 GEMVs (sbvr_gemv_ex AUTO)
    sbvr_gemv_problem pr = {};
    pr.w = *w;
    const size_t e = group_workspace_bytes(&pr, 1);
    if (e > *bytes) *bytes = e;
  }
  return SBVR_OK;
}

sbvr_status sbvr_workspace_init(void* workspace, size_t bytes, void* stream) {
  if (!workspace && bytes) return set_error(SBVR_ERR_INVALID_ARG, "workspace is NULL");
  if (bytes == 0) return SBVR_OK;
  cudaError_t e = cudaMemsetAsync(workspace, 0xFF, bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  return SBVR_OK;
}

sbvr_status sbvr_gemv_ex(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* Y, void* workspace,
                         size_t ws_bytes, int32_t algo, void* stream) {
  sbvr_status s = check_weights(w);
  if (s != SBVR_OK) return s;
  s = check_act(w, X, T);
  if (s != SBVR_OK) return s;
  if (!Y) return set_error(SBVR_ERR_INVALID_ARG, "Y is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (X->kind == SBVR_ACT_FP16_Q) {
    if (algo != SBVR_ALGO_AUTO && algo != SBVR_ALGO_MMA)
      return set_error(SBVR_ERR_UNSUPPORTED, "in-kernel conversion runs on the MMA kernel, not algo %d", algo);
    size_t need = mma_workspace_bytes(w, T);
    if (need && (!workspace || ws_bytes < need))
      return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return launch_gemv_mma(w, X, T, Y, workspace, ws_bytes, nullptr, st);
  }
  if (w->meta_kind == SBVR_META_INDEXED) {
    // table + index weights: the mma.sync kernel (every SBVR-x form), K 2..4
    if (X->kind != SBVR_ACT_SBVR) return set_error(SBVR_ERR_UNSUPPORTED, "indexed weights need an SBVR-x activation");
    if (w->K < 2 || w->K > 4) return set_error(SBVR_ERR_UNSUPPORTED, "indexed weights: K=%d outside 2..4", w->K);
    if (algo != SBVR_ALGO_AUTO && algo != SBVR_ALGO_MMA)
      return set_error(SBVR_ERR_UNSUPPORTED, "indexed weights run on the MMA kernel, not algo %d", algo);
    size_t need = mma_workspace_bytes(w, T);
    if (need && (!workspace || ws_bytes < need))
      return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return launch_gemv_mma(w, X, T, Y, workspace, ws_bytes, nullptr, st);
  }
  if (X->kind == SBVR_ACT_FP16) {
    // fp16-x: MMA (mma.m16n8k16 f16, tokens as MMA columns) by default; POPC selects the CUDA-core
    // reference kernel (one predicated add per set bit)
    if (algo == SBVR_ALGO_POPC) return launch_gemv_fp16x(w, X, T, Y, st);
    if (algo != SBVR_ALGO_AUTO && algo != SBVR_ALGO_MMA)
      return set_error(SBVR_ERR_UNSUPPORTED, "fp16-x runs on the MMA (default) or POPC kernel, not algo %d", algo);
    size_t need = mma_workspace_bytes(w, T);
    if (need && (!workspace || ws_bytes < need))
      return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return launch_gemv_mma(w, X, T, Y, workspace, ws_bytes, nullptr, st);
  }
  // diagnostics only (A/B timing in tools/): SBVR_FORCE_ALGO=<sbvr_algo> overrides AUTO for SBVR-x
  static const int forced = getenv("SBVR_FORCE_ALGO") ? atoi(getenv("SBVR_FORCE_ALGO")) : 0;
  if (algo == SBVR_ALGO_AUTO) {
    if (forced > 0 && forced <= SBVR_ALGO_ZT && !(forced == SBVR_ALGO_PIPE && T != 1)) algo = forced;
  }
  if (algo == SBVR_ALGO_POPC) return launch_gemv_popc(w, X, T, Y, nullptr, st);
  if (algo == SBVR_ALGO_AUTO) {
    // batch 1 on a large matrix (>= 2^26 weights, e.g. a 70B MLP projection): the grouped kernel with one problem
    // (whole 128-row unit records, one copy per warp pair; measured 4-7 % faster there, slower on small shapes)
    if (T == 1 && !forced && w->meta_kind == SBVR_META_GROUP && w->K >= 2 && w->K <= 4 && w->M % kRowBlock == 0 &&
        (long)w->M * w->N >= (1L << 26)) {
      sbvr_gemv_problem pr;
      pr.w = *w;
      pr.x = *X;
      pr.y = Y;
      const size_t need = group_workspace_bytes(&pr, 1);
      if (workspace && ws_bytes >= need) return launch_gemv_group(&pr, 1, workspace, ws_bytes, st);
    }
    // batches: the tcgen05 z-column kernel (one weight pass per 32 tokens) from zt_min tokens on; batch 1-2:
    // the mma.sync bit-plane kernel.  SBVR_ZT_MIN_T overrides the switch point (A/B timing).
    static const int zt_min = getenv("SBVR_ZT_MIN_T") ? atoi(getenv("SBVR_ZT_MIN_T")) : 12;
    algo = (T >= zt_min && zt_supported(w, X)) ? SBVR_ALGO_ZT : SBVR_ALGO_MMA;
  }
  if (algo == SBVR_ALGO_ZT) {
    if (!zt_supported(w, X)) return set_error(SBVR_ERR_UNSUPPORTED, "ZT needs an SBVR-x activation and K <= 4 (K=%d)", w->K);
    size_t need = zt_workspace_bytes(w, T);
    if (!workspace || ws_bytes < need)
      return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return launch_gemv_zt(w, X, T, Y, workspace, ws_bytes, nullptr, st);
  }
  if (algo == SBVR_ALGO_PIPE) {
    if (T != 1) return set_error(SBVR_ERR_UNSUPPORTED, "PIPE runs batch 1 (T=%d)", T);
    size_t need = pipe_workspace_bytes(w);
    if (!workspace || ws_bytes < need)
      return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return launch_gemv_pipe(w, X, Y, workspace, nullptr, st);
  }
  if (algo != SBVR_ALGO_TC && algo != SBVR_ALGO_MMA) return set_error(SBVR_ERR_INVALID_ARG, "bad algo %d", algo);
  size_t need = algo == SBVR_ALGO_TC ? tc_workspace_bytes(w, T) : mma_workspace_bytes(w, T);
  if (need && (!workspace || ws_bytes < need))
    return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
  if (algo == SBVR_ALGO_TC) return launch_gemv_tc(w, X, T, Y, workspace, ws_bytes, nullptr, st);
  return launch_gemv_mma(w, X, T, Y, workspace, ws_bytes, nullptr, st);
}

sbvr_status sbvr_gemv(const sbvr_weights* w, const sbvr_act* x, float* y, void* workspace, size_t ws_bytes,
                      void* stream) {
  return sbvr_gemv_ex(w, x, 1, y, workspace, ws_bytes, SBVR_ALGO_AUTO, stream);
}

sbvr_status sbvr_gemv_chain(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* Y, void* workspace,
                            size_t ws_bytes, const sbvr_weights* next_w, void* stream) {
  if (!next_w) return sbvr_gemv_batched(w, X, T, Y, workspace, ws_bytes, stream);
  sbvr_status s = check_weights(next_w);
  if (s != SBVR_OK) return s;
  s = check_weights(w);
  if (s != SBVR_OK) return s;
  s = check_act(w, X, T);
  if (s != SBVR_OK) return s;
  if (!Y) return set_error(SBVR_ERR_INVALID_ARG, "Y is NULL");
  // the hint is honoured by the mma.sync kernel (batch 1-2 and its batched forms); elsewhere it is ignored
  const bool mma = (X->kind == SBVR_ACT_SBVR || X->kind == SBVR_ACT_FP16_Q) &&
                   (w->meta_kind == SBVR_META_INDEXED ? (w->K >= 2 && w->K <= 4) : true);
  static const int zt_min = getenv("SBVR_ZT_MIN_T") ? atoi(getenv("SBVR_ZT_MIN_T")) : 12;
  if (!mma || (w->meta_kind == SBVR_META_GROUP && T >= zt_min && zt_supported(w, X)))
    return sbvr_gemv_batched(w, X, T, Y, workspace, ws_bytes, stream);
  size_t need = mma_workspace_bytes(w, T);
  if (need && (!workspace || ws_bytes < need))
    return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
  return launch_gemv_mma(w, X, T, Y, workspace, ws_bytes, nullptr, (cudaStream_t)stream, nullptr, next_w);
}

sbvr_status sbvr_gemv_to_peers(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* const* peer_y,
                               int32_t n_peers, int32_t y_row_offset, int32_t M_full, void* workspace, size_t ws_bytes,
                               void* stream) {
  sbvr_status s = check_weights(w);
  if (s != SBVR_OK) return s;
  s = check_act(w, X, T);
  if (s != SBVR_OK) return s;
  if (!peer_y) return set_error(SBVR_ERR_INVALID_ARG, "peer_y is NULL");
  if (w->meta_kind == SBVR_META_INDEXED && (X->kind == SBVR_ACT_FP16 || w->K < 2 || w->K > 4))
    return set_error(SBVR_ERR_UNSUPPORTED, "indexed weights need SBVR-x and K 2..4");
  if (n_peers < 1 || n_peers > 8) return set_error(SBVR_ERR_INVALID_ARG, "n_peers=%d outside 1..8", n_peers);
  if (y_row_offset < 0 || M_full < w->M || y_row_offset > M_full - w->M)
    return set_error(SBVR_ERR_SHAPE, "rows [%d, %d) do not fit M_full=%d", y_row_offset, y_row_offset + w->M, M_full);
  PeerOut po;
  po.n = n_peers;
  po.row_offset = y_row_offset;
  po.M_full = M_full;
  for (int j = 0; j < 8; ++j) {
    po.y[j] = j < n_peers ? peer_y[j] : nullptr;
    if (j < n_peers && !po.y[j]) return set_error(SBVR_ERR_INVALID_ARG, "peer_y[%d] is NULL", j);
  }
  size_t need = mma_workspace_bytes(w, T);
  if (need && (!workspace || ws_bytes < need))
    return set_error(SBVR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
  return launch_gemv_mma(w, X, T, nullptr, workspace, ws_bytes, nullptr, (cudaStream_t)stream, &po);
}

static sbvr_status check_group(const sbvr_gemv_problem* probs, int32_t n) {
  if (!probs) return set_error(SBVR_ERR_INVALID_ARG, "probs is NULL");
  if (n < 1 || n > SBVR_GROUP_MAX) return set_error(SBVR_ERR_INVALID_ARG, "n=%d outside 1..%d", n, SBVR_GROUP_MAX);
  for (int i = 0; i < n; ++i) {
    const sbvr_gemv_problem& p = probs[i];
    sbvr_status s = check_weights(&p.w);
    if (s != SBVR_OK) return s;
    s = check_act(&p.w, &p.x, 1);
    if (s != SBVR_OK) return s;
    if (!p.y) return set_error(SBVR_ERR_INVALID_ARG, "problem %d: y is NULL", i);
    if (p.x.kind != SBVR_ACT_SBVR && p.x.kind != SBVR_ACT_FP16_Q)
      return set_error(SBVR_ERR_UNSUPPORTED, "problem %d: grouped GEMV needs SBVR-x or SBVR_ACT_FP16_Q", i);
    if (p.x.kind != probs[0].x.kind)
      return set_error(SBVR_ERR_UNSUPPORTED, "problem %d: activation kind differs from problem 0", i);
    if (p.w.meta_kind != SBVR_META_GROUP)
      return set_error(SBVR_ERR_UNSUPPORTED, "problem %d: grouped GEMV needs SBVR_META_GROUP weights", i);
    if (p.w.K < 2 || p.w.K > 4) return set_error(SBVR_ERR_UNSUPPORTED, "problem %d: K=%d outside 2..4", i, p.w.K);
    if (p.w.K != probs[0].w.K) return set_error(SBVR_ERR_UNSUPPORTED, "problem %d: K differs from problem 0", i);
    if (p.x.l != probs[0].x.l) return set_error(SBVR_ERR_UNSUPPORTED, "problem %d: l differs from problem 0", i);
    if (p.w.M % kRowBlock) return set_error(SBVR_ERR_SHAPE, "problem %d: M=%d not a multiple of 128", i, p.w.M);
  }
  return SBVR_OK;
}

sbvr_status sbvr_gemv_group_workspace_bytes(const sbvr_gemv_problem* probs, int32_t n, size_t* bytes) {
  if (!bytes) return set_error(SBVR_ERR_INVALID_ARG, "bytes is NULL");
  if (!probs || n < 1 || n > SBVR_GROUP_MAX) return set_error(SBVR_ERR_INVALID_ARG, "probs/n invalid");
  for (int i = 0; i < n; ++i)
    if (probs[i].w.M <= 0 || probs[i].w.N <= 0 || probs[i].w.M % kRowBlock || probs[i].w.N % kG)
      return set_error(SBVR_ERR_SHAPE, "problem %d: bad M/N %d/%d", i, probs[i].w.M, probs[i].w.N);
  *bytes = group_workspace_bytes(probs, n);
  return SBVR_OK;
}

sbvr_status sbvr_gemv_group_to_peers(const sbvr_gemv_problem* probs, int32_t n, float* const* peer_y, int32_t n_peers,
                                     const int32_t* y_row_offset, const int32_t* M_full, void* workspace,
                                     size_t ws_bytes, void* stream) {
  if (!peer_y || !y_row_offset || !M_full) return set_error(SBVR_ERR_INVALID_ARG, "peer_y / offsets / M_full is NULL");
  if (n_peers < 1 || n_peers > 8) return set_error(SBVR_ERR_INVALID_ARG, "n_peers=%d outside 1..8", n_peers);
  if (!probs || n < 1 || n > SBVR_GROUP_MAX) return set_error(SBVR_ERR_INVALID_ARG, "probs/n invalid");
  // probs[i].y is not used: validate with a stand-in so check_group accepts the descriptors
  sbvr_gemv_problem tmp[SBVR_GROUP_MAX];
  for (int i = 0; i < n; ++i) {
    tmp[i] = probs[i];
    tmp[i].y = peer_y[i * n_peers];
    if (y_row_offset[i] < 0 || M_full[i] < probs[i].w.M || y_row_offset[i] > M_full[i] - probs[i].w.M)
      return set_error(SBVR_ERR_SHAPE, "problem %d: rows [%d, %d) do not fit M_full=%d", i, y_row_offset[i],
                       y_row_offset[i] + probs[i].w.M, M_full[i]);
    for (int j = 0; j < n_peers; ++j)
      if (!peer_y[i * n_peers + j]) return set_error(SBVR_ERR_INVALID_ARG, "peer_y[%d][%d] is NULL", i, j);
  }
  sbvr_status s = check_group(tmp, n);
  if (s != SBVR_OK) return s;
  if (!workspace) return set_error(SBVR_ERR_WORKSPACE, "workspace is NULL");
  GroupPeers gp;
  gp.y = peer_y;
  gp.n = n_peers;
  gp.row_offset = y_row_offset;
  return launch_gemv_group(tmp, n, workspace, ws_bytes, (cudaStream_t)stream, &gp);
}

sbvr_status sbvr_gemv_group(const sbvr_gemv_problem* probs, int32_t n, void* workspace, size_t ws_bytes, void* stream) {
  sbvr_status s = check_group(probs, n);
  if (s != SBVR_OK) return s;
  if (!workspace) return set_error(SBVR_ERR_WORKSPACE, "workspace is NULL");
  return launch_gemv_group(probs, n, workspace, ws_bytes, (cudaStream_t)stream);
}

sbvr_status sbvr_gemv_batched(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* Y, void* workspace,
                              size_t ws_bytes, void* stream) {
  return sbvr_gemv_ex(w, X, T, Y, workspace, ws_bytes, SBVR_ALGO_AUTO, stream);
}

sbvr_status sbvr_hadamard_rows(const void* X, void* Y, int32_t dtype, int32_t rows, int32_t N, int32_t block,
                               const int8_t* signs, void* stream) {
  if (!X || !Y || !signs) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  if (dtype != SBVR_F32 && dtype != SBVR_F16) return set_error(SBVR_ERR_UNSUPPORTED, "dtype %d (F32 or F16)", dtype);
  if (block < 32 || block > 1024 || (block & (block - 1)))
    return set_error(SBVR_ERR_UNSUPPORTED, "block %d: a power of two in 32..1024", block);
  if (rows < 0 || N <= 0 || N % block) return set_error(SBVR_ERR_SHAPE, "rows=%d N=%d block=%d", rows, N, block);
  if (!aligned16(X) || !aligned16(Y)) return set_error(SBVR_ERR_ALIGNMENT, "X/Y must be 16-byte aligned");
  return launch_hadamard(X, Y, dtype, rows, N, block, signs, (cudaStream_t)stream);
}

sbvr_status sbvr_debug_partials(const sbvr_weights* w, const sbvr_act* x, int32_t algo, int32_t* P, void* stream) {
  sbvr_status s = check_weights(w);
  if (s != SBVR_OK) return s;
  s = check_act(w, x, 1);
  if (s != SBVR_OK) return s;
  if (!P) return set_error(SBVR_ERR_INVALID_ARG, "P is NULL");
  if (x->kind != SBVR_ACT_SBVR) return set_error(SBVR_ERR_INVALID_ARG, "partials need an SBVR activation");
  if (w->meta_kind == SBVR_META_INDEXED && algo != SBVR_ALGO_MMA && algo != SBVR_ALGO_AUTO)
    return set_error(SBVR_ERR_UNSUPPORTED, "indexed weights run on the MMA kernel");
  if (w->meta_kind == SBVR_META_INDEXED && (w->K < 2 || w->K > 4))
    return set_error(SBVR_ERR_UNSUPPORTED, "indexed weights: K=%d outside 2..4", w->K);
  if (algo == SBVR_ALGO_POPC) return launch_gemv_popc(w, x, 1, nullptr, P, (cudaStream_t)stream);
  if (algo == SBVR_ALGO_TC) return launch_gemv_tc(w, x, 1, nullptr, nullptr, 0, P, (cudaStream_t)stream);
  if (algo == SBVR_ALGO_MMA || algo == SBVR_ALGO_AUTO)
    return launch_gemv_mma(w, x, 1, nullptr, nullptr, 0, P, (cudaStream_t)stream);
  if (algo == SBVR_ALGO_PIPE) return launch_gemv_pipe(w, x, nullptr, nullptr, P, (cudaStream_t)stream);
  return set_error(SBVR_ERR_INVALID_ARG, "bad algo %d", algo);
}

static sbvr_status check_prefill(const sbvr_weights* w, int32_t T) {
  sbvr_status s = check_weights(w);
  if (s != SBVR_OK) return s;
  if (w->meta_kind != SBVR_META_GROUP)
    return set_error(SBVR_ERR_UNSUPPORTED, "prefill reads SBVR_META_GROUP weights (decompress indexed weights' table)");
  if (w->K < 1 || w->K > 4) return set_error(SBVR_ERR_UNSUPPORTED, "prefill: K=%d (1..4)", w->K);
  if (T < 0) return set_error(SBVR_ERR_SHAPE, "T=%d", T);
  return SBVR_OK;
}

sbvr_status sbvr_prefill_workspace_bytes(const sbvr_weights* w, int32_t T, size_t* bytes) {
  sbvr_status s = check_prefill(w, T);
  if (s != SBVR_OK) return s;
  if (!bytes) return set_error(SBVR_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = T > 0 ? prefill_workspace_bytes(w, T) : 0;
  return SBVR_OK;
}

sbvr_status sbvr_prefill(const sbvr_weights* w, const uint16_t* X, int32_t T, float* Y, void* workspace,
                         size_t ws_bytes, void* stream) {
  sbvr_status s = check_prefill(w, T);
  if (s != SBVR_OK) return s;
  if (T == 0) return SBVR_OK;
  if (!X || !Y) return set_error(SBVR_ERR_INVALID_ARG, "X or Y is NULL");
  if ((reinterpret_cast<uintptr_t>(X) & 7) || (reinterpret_cast<uintptr_t>(Y) & 3))
    return set_error(SBVR_ERR_ALIGNMENT, "X must be 8-byte and Y 4-byte aligned");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return set_error(workspace ? SBVR_ERR_ALIGNMENT : SBVR_ERR_WORKSPACE, "workspace NULL or not 256-byte aligned");
  return launch_prefill(w, X, T, Y, workspace, ws_bytes, (cudaStream_t)stream);
}

sbvr_status sbvr_debug_zt_sums(const sbvr_weights* w, const sbvr_act* x, int32_t T, int32_t* Tsum, void* stream) {
  sbvr_status s = check_weights(w);
  if (s != SBVR_OK) return s;
  s = check_act(w, x, T);
  if (s != SBVR_OK) return s;
  if (!Tsum) return set_error(SBVR_ERR_INVALID_ARG, "Tsum is NULL");
  if (w->meta_kind != SBVR_META_GROUP) return set_error(SBVR_ERR_UNSUPPORTED, "ZT reads SBVR_META_GROUP weights");
  if (T > 32) return set_error(SBVR_ERR_SHAPE, "T=%d: the debug export covers one pass (T <= 32)", T);
  if (!zt_supported(w, x)) return set_error(SBVR_ERR_UNSUPPORTED, "ZT needs SBVR-x and K <= 4");
  return launch_gemv_zt(w, x, T, nullptr, nullptr, 0, Tsum, (cudaStream_t)stream);
}

static sbvr_status check_pack_args(int32_t M, int32_t N, int32_t K, int32_t G) {
  if (G != kG) return set_error(SBVR_ERR_UNSUPPORTED, "group_size %d (only 128)", G);
  if (K < 1 || K > kMaxK) return set_error(SBVR_ERR_UNSUPPORTED, "K=%d", K);
  if (M <= 0 || N <= 0 || M % kTileRows || N % kG) return set_error(SBVR_ERR_SHAPE, "M=%d N=%d", M, N);
  return SBVR_OK;
}

sbvr_status sbvr_pack_canonical(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint32_t* planes_canon,
                                const uint16_t* s16, const uint16_t* b16, const uint8_t* r_idx, uint8_t* data) {
  sbvr_status s = check_pack_args(M, N, K, group_size);
  if (s != SBVR_OK) return s;
  if (!planes_canon || !s16 || !b16 || !r_idx || !data) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  Layout Lo(M, N, K);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < Lo.NG; ++g) {
      long q = (long)r * Lo.NG + g;
      for (int t = 0; t < K; ++t)
        for (int c = 0; c < kWPG; ++c)
          memcpy(data + Lo.plane_byte(r, g, t, c), planes_canon + (q * K + t) * kWPG + c, 4);
      const uint32_t sb = (uint32_t)s16[q] | ((uint32_t)b16[q] << 16);
      memcpy(data + Lo.sb_byte(r, g), &sb, 4);
      data[Lo.ri_byte(r, g)] = r_idx[q];
    }
  return SBVR_OK;
}

sbvr_status sbvr_unpack_canonical(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint8_t* data,
                                  uint32_t* planes_canon, uint16_t* s16, uint16_t* b16, uint8_t* r_idx) {
  sbvr_status s = check_pack_args(M, N, K, group_size);
  if (s != SBVR_OK) return s;
  if (!planes_canon || !s16 || !b16 || !r_idx || !data) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  Layout Lo(M, N, K);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < Lo.NG; ++g) {
      long q = (long)r * Lo.NG + g;
      for (int t = 0; t < K; ++t)
        for (int c = 0; c < kWPG; ++c)
          memcpy(planes_canon + (q * K + t) * kWPG + c, data + Lo.plane_byte(r, g, t, c), 4);
      uint32_t sb;
      memcpy(&sb, data + Lo.sb_byte(r, g), 4);
      s16[q] = (uint16_t)(sb & 0xffffu);
      b16[q] = (uint16_t)(sb >> 16);
      r_idx[q] = data[Lo.ri_byte(r, g)];
    }
  return SBVR_OK;
}

sbvr_status sbvr_pack_indexed(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint32_t* planes_canon,
                              const uint8_t* idx, uint8_t* data) {
  sbvr_status s = check_pack_args(M, N, K, group_size);
  if (s != SBVR_OK) return s;
  if (!planes_canon || !idx || !data) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  IdxLayout Lo(M, N, K);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < Lo.NG; ++g) {
      long q = (long)r * Lo.NG + g;
      for (int t = 0; t < K; ++t)
        for (int c = 0; c < kWPG; ++c) memcpy(data + Lo.plane_byte(r, g, t, c), planes_canon + (q * K + t) * kWPG + c, 4);
      data[Lo.idx_byte(r, g)] = idx[q];
    }
  return SBVR_OK;
}

sbvr_status sbvr_unpack_indexed(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint8_t* data,
                                uint32_t* planes_canon, uint8_t* idx) {
  sbvr_status s = check_pack_args(M, N, K, group_size);
  if (s != SBVR_OK) return s;
  if (!planes_canon || !idx || !data) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  IdxLayout Lo(M, N, K);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < Lo.NG; ++g) {
      long q = (long)r * Lo.NG + g;
      for (int t = 0; t < K; ++t)
        for (int c = 0; c < kWPG; ++c) memcpy(planes_canon + (q * K + t) * kWPG + c, data + Lo.plane_byte(r, g, t, c), 4);
      idx[q] = data[Lo.idx_byte(r, g)];
    }
  return SBVR_OK;
}

sbvr_status sbvr_fill_ratio_table(const sbvr_weights* w, void* stream) {
  if (!w || !w->ratio_pow) return set_error(SBVR_ERR_INVALID_ARG, "NULL pointer");
  if (w->K < 1 || w->K > kMaxK) return set_error(SBVR_ERR_UNSUPPORTED, "K=%d", w->K);
  if (w->n_ratio < 2 || w->n_ratio > 64 || (w->n_ratio & 1)) return set_error(SBVR_ERR_INVALID_ARG, "n_ratio");
  return launch_ratio_table(w->ratio_pow, w->n_ratio, w->K, (cudaStream_t)stream);
}

}  // extern "C"
