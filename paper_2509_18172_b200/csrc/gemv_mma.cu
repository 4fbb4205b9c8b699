// gemv_mma.cu -- host side of the mma.sync SBVR GEMV (kernel: gemv_mma.cuh): work partition, workspace,
// pass splitting over tokens, dispatch to the per-K instantiations (gemv_mma_k<K>.cu).
#include "gemv_mma.cuh"

namespace sbvr {
namespace mma {
extern template cudaError_t launch_k<1>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<2>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<3>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<4>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<5>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<6>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<7>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
extern template cudaError_t launch_k<8>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
}  // namespace mma

using namespace mma;
namespace {

static int num_sms() {
  // per device: a process may drive several GPUs
  static int n[64] = {0};
  const int dev = cur_device();
  if (dev < 0 || dev >= 64) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

struct Plan {
  int NG, MT, n_full, tail_nb, n_bands;
  int Us_main, C_main, Us_tail, C_tail;
};

// CTAs per launch: one per SM (16 warps; every SM gets the same work, and a CTA of the next
// launch cannot co-reside and idle at griddepcontrol.wait while holding half an SM), at most one
// per kMinUnitsPerCta units.
static int ctas_for(int Us, int NG) {
  if (Us <= 0) return 0;
  int C = num_sms() * SBVR_MMA_CTAS_PER_SM;
  const int cap = (Us + kMinUnitsPerCta - 1) / kMinUnitsPerCta;
  if (C > cap) C = cap;
  return C < 1 ? 1 : C;
}

static Plan make_plan(const sbvr_weights* w) {
  Plan pl;
  pl.NG = w->N / kG;
  pl.MT = w->M / kTileRows;
  pl.n_full = pl.MT / 4;
  pl.tail_nb = pl.MT % 4;
  pl.n_bands = pl.n_full + (pl.tail_nb ? 1 : 0);
  pl.Us_main = pl.n_full * pl.NG;
  pl.C_main = ctas_for(pl.Us_main, pl.NG);
  pl.Us_tail = pl.tail_nb ? pl.NG : 0;
  pl.C_tail = ctas_for(pl.Us_tail, pl.NG);
  return pl;
}

// workspace = [band arrival counters (u32, one per 64-row band), padded to 256 B]
//             [partials: CTA x {first, last band} x 8 token columns x 64 rows fp32]
// (sized for the widest pass, TT = 8, whatever T is; all 0xFF at rest -- sbvr_workspace_init)
static size_t mma_cnt_bytes(const Plan& pl) { return ((size_t)(pl.n_bands + 1) * 4 + 255) / 256 * 256; }

size_t mma_workspace_bytes_(const sbvr_weights* w, int /*T*/) {
  const Plan pl = make_plan(w);
  const int C = pl.C_main > pl.C_tail ? pl.C_main : pl.C_tail;
  return mma_cnt_bytes(pl) + (size_t)C * 2 * 8 * 64 * sizeof(float);
}

static cudaError_t launch_any(int K, const ImmaParams& p, int NB, int TT, bool debug, bool f16x, bool zb, cudaStream_t st) {
  switch (K) {
    case 1: return launch_k<1>(p, NB, TT, debug, f16x, zb, st);
    case 2: return launch_k<2>(p, NB, TT, debug, f16x, zb, st);
    case 3: return launch_k<3>(p, NB, TT, debug, f16x, zb, st);
    case 4: return launch_k<4>(p, NB, TT, debug, f16x, zb, st);
    case 5: return launch_k<5>(p, NB, TT, debug, f16x, zb, st);
    case 6: return launch_k<6>(p, NB, TT, debug, f16x, zb, st);
    case 7: return launch_k<7>(p, NB, TT, debug, f16x, zb, st);
    default: return launch_k<8>(p, NB, TT, debug, f16x, zb, st);
  }
}

}  // namespace

size_t mma_workspace_bytes(const sbvr_weights* w, int T) { return mma_workspace_bytes_(w, T); }

sbvr_status launch_gemv_mma(const sbvr_weights* w, const sbvr_act* x, int T, float* Y, void* ws, size_t ws_bytes,
                            int32_t* P_debug, cudaStream_t st, const PeerOut* peers, const sbvr_weights* next_w) {
  const Plan pl = make_plan(w);
  ImmaParams p;
  p.nx_units = nullptr;
  if (next_w && next_w->meta_kind == SBVR_META_GROUP) {
    const Plan nx = make_plan(next_w);
    if (nx.Us_main > 0) {
      p.nx_units = next_w->data;
      p.nx_NG = nx.NG;
      p.nx_K = next_w->K;
      p.nx_Us = nx.Us_main;
      p.nx_C = nx.C_main;
      p.nx_qq = nx.Us_main / nx.C_main;
      p.nx_rr = nx.Us_main % nx.C_main;
    }
  }
  p.n_peers = peers ? peers->n : 0;
  p.y_off = peers ? peers->row_offset : 0;
  p.M_full = peers ? peers->M_full : w->M;
  for (int j = 0; j < 8; ++j) p.peer_y[j] = peers && j < peers->n ? peers->y[j] : nullptr;
  p.ratio_pow = w->ratio_pow;
  p.coef_table = w->meta_kind == SBVR_META_INDEXED ? w->coef_table : nullptr;
  p.units = w->data;
  p.K = w->K;
  p.n_full = w->M / kRowBlock;
  p.tail_rows = w->M % kRowBlock;
  p.M = w->M; p.N = w->N; p.l = x->l; p.n_ratio = w->n_ratio;
  p.P = P_debug;
  p.one = 1;
  {
    const char* em = getenv("SBVR_EXP_MODE");
    p.exp = em ? atoi(em) : 0;
    const char* tsp = getenv("SBVR_TS_PTR");
    p.ts = tsp ? reinterpret_cast<unsigned long long*>(strtoull(tsp, nullptr, 0)) : nullptr;
  }
  if (!P_debug && ws_bytes < mma_workspace_bytes_(w, T))
    return set_error(SBVR_ERR_WORKSPACE, "gemv_mma: workspace %zu bytes < required %zu", ws_bytes,
                     mma_workspace_bytes_(w, T));
  p.ws_cnt = ws ? reinterpret_cast<unsigned int*>(ws) : nullptr;
  p.ws_part = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + mma_cnt_bytes(pl)) : nullptr;
  const bool f16x = x->kind == SBVR_ACT_FP16;
  const bool xq = x->kind == SBVR_ACT_FP16_Q;     // fp16 x, converted to SBVR-x in the kernel prologue (T = 1)
  const uint32_t* xp = (f16x || xq) ? nullptr : static_cast<const uint32_t*>(x->data);
  const uint16_t* xh = f16x ? static_cast<const uint16_t*>(x->data) : nullptr;
  p.xq = xq ? static_cast<const uint16_t*>(x->data) : nullptr;
  p.xq_groups = 0;
  const bool debug = P_debug != nullptr;
  // SBVR-x batches: tokens as MMA columns, B = z (s8), A = the plane bits themselves (u8 0/1); one pass
  // serves 8 tokens with T_t = sum_e beta_t[e] z_e read directly from the accumulator
  static const int zb_min = getenv("SBVR_ZB_MIN_T") ? atoi(getenv("SBVR_ZB_MIN_T")) : kZbMinT;
  const bool zb = !f16x && !debug && T >= zb_min;
  int done = 0;
  while (done < T) {
    const int rem = T - done;
    int TT;
    if (f16x || zb) TT = (zb || rem > 4) ? 8 : (rem > 2 ? 4 : rem);   // token columns of the MMA
    else TT = debug ? 1 : (rem >= 4 ? 4 : (rem >= 2 ? 2 : 1));
    const int ntok = rem < TT ? rem : TT;
    p.ntok = ntok;
    p.xplanes = (f16x || xq) ? nullptr : xp + (size_t)done * pl.NG * x->l * 4;
    p.xscales = (f16x || xq) ? nullptr : x->scales + (size_t)done * pl.NG;
    p.xh = f16x ? xh + (size_t)done * w->N : nullptr;
    p.Y = Y ? Y + (size_t)done * w->M : nullptr;
    for (int j = 0; j < p.n_peers; ++j) p.peer_y[j] = peers->y[j] + (size_t)done * p.M_full;
    for (int part = 0; part < 2; ++part) {
      const int NB = part == 0 ? 4 : pl.tail_nb;
      const int Us = part == 0 ? pl.Us_main : pl.Us_tail;
      if (Us == 0) continue;
      p.band0 = part == 0 ? 0 : pl.n_full;
      p.Us = Us;
      p.Pw = part == 0 ? pl.C_main : pl.C_tail;
      p.qq = Us / p.Pw;
      p.rr = Us % p.Pw;
      if (xq) p.xq_groups = p.qq + (p.rr ? 1 : 0) < pl.NG ? p.qq + (p.rr ? 1 : 0) : pl.NG;
      // balance warp ranges at tile granularity: an extra tile pair on some warps costs a whole pair
      // step at the end of a launch, a lone tile half of it (measured on the bench step: +0.7 %, the
      // big GEMVs 1.5 % faster; a pair-granular split for small problems measured no better)
      p.fine = 1;
      const uint8_t* nx_keep = p.nx_units;
      if (part != 0 || done + ntok < T) p.nx_units = nullptr;     // the hint belongs to the last pass, main launch
      cudaError_t e = launch_any(w->K, p, NB, TT, debug, f16x, zb, st);
      p.nx_units = nx_keep;
      if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "gemv_mma setup: %s", cudaGetErrorString(e));
      sbvr_status s = check_launch("gemv_mma_kernel");
      if (s != SBVR_OK) return s;
    }
    if (debug) break;
    done += ntok;
  }
  return SBVR_OK;
}

}  // namespace sbvr

