// encode_weights.cu -- offline SBVR weight encoding, §4.2, strict fp64.
//
// One CTA per weight group (groups are independent, "grouping facilitates parallelism
// during the encoding step"):
//   1. load the 128 values as fp64 (exact from fp32/fp16/bf16), bitonic-sort a copy in smem;
//      thread 0 derives q95 (linear interpolation, reading A6), min, max and the mean
//      (sequential sum in element order) -> s_min, s_max, s_gran, b_max, b_gran (Eq. 8-11);
//   2. S (Eq. 6) and B (Eq. 7) candidates rounded to fp16 (reading A15), R as two linspaces
//      over [-1,-0.5] and [0.5,1] (reading A3);
//   3. Algorithm 1: thread t scans entries e = t, t+256, ... (R outer, S middle,
//      B inner): c = s r^t + b (Eq. 4), 2^K subset sums, per element the distance to the
//      nearest sum (min over all sums), SSE in element order, mse = SSE/128; strict '<' keeps
//      the first best; a CTA arg-min (mse, then entry index) equals the sequential scan;
//   4. P:231 bit assignment for the winner (ties: smaller value, then smaller mask, reading A8),
//      __ballot_sync packs each 32-element word of each plane; write planes / meta / mse.
// Every fp64 operation is an explicit _rn intrinsic in the order the paper's formulas are
// written, so the result is bit-identical to any IEEE fp64 evaluation in that order.
#include <cfloat>

#include "sbvr_internal.cuh"

namespace sbvr {

__device__ __forceinline__ uint16_t f64_to_f16_bits(double x) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}
__device__ __forceinline__ double f16_bits_to_f64(uint16_t h) {
  float f;
  asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
  return (double)f;
}

__device__ __forceinline__ double ratio_value(int i, int n_ratio) {
  const int half = n_ratio / 2;
  const int part = i / half, ii = i % half;
  const double a = part ? 0.5 : -1.0;
  const double b = part ? 1.0 : -0.5;
  if (half == 1) return a;
  if (ii == half - 1) return b;
  return __dadd_rn(__dmul_rn((double)ii, __ddiv_rn(__dsub_rn(b, a), (double)(half - 1))), a);
}

__device__ __forceinline__ double load_w(const void* W, int dtype, size_t idx) {
  if (dtype == SBVR_F32) return (double)__ldg(reinterpret_cast<const float*>(W) + idx);
  const unsigned short u = __ldg(reinterpret_cast<const unsigned short*>(W) + idx);
  if (dtype == SBVR_F16) return (double)__half2float(__ushort_as_half(u));
  return (double)__uint_as_float(((uint32_t)u) << 16);  // bf16
}

struct EncParams {
  const void* W;
  int dtype, M, N;
  int n_ratio, n_scale, n_bias;
  double s_min_factor;
  uint8_t* data;
  double* group_mse;
  uint8_t* group_hit;     // cached encoder: 1 = the group took a cached coefficient set
  int fast;               // 1: fp32 search of every entry, fp64 (strict) re-evaluation of the near-best ones
  int m32_cap;            // fast mode: entries whose fp32 MSE fits in dynamic shared memory
  int cache_size;         // cached encoder: MRU capacity (0..64)
  double cache_alpha;     // cached encoder: moving-average weight
};

// Shared-memory state of one CTA encoding one group at a time.
struct GroupSmem {
  double* X;      // [128] group values (element order)
  double* Xs;     // [128] sorted copy
  double* R;      // [n_ratio]
  double* S;      // [n_scale]
  double* B;      // [n_bias]
};

__device__ __forceinline__ void grp_load(const EncParams& p, const GroupSmem& sm, int row, int g) {
  const int tid = threadIdx.x;
  if (tid < kG) {
    const double v = load_w(p.W, p.dtype, (size_t)row * p.N + (size_t)g * kG + tid);
    sm.X[tid] = v;
    sm.Xs[tid] = v;
  }
}

// O-W1 statistics + O-W2 candidate sets (Eq. 5-11) into sm.S, sm.B.  Call with all threads.
template <int K>
__device__ void grp_candidates(const EncParams& p, const GroupSmem& sm, double* s_scal) {
  const int tid = threadIdx.x;
  __syncthreads();
  // bitonic sort of Xs (ascending); any correct sort yields the same array
  for (int k2 = 2; k2 <= kG; k2 <<= 1) {
    for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
      if (tid < kG) {
        const int ixj = tid ^ j2;
        if (ixj > tid) {
          const double a = sm.Xs[tid], b = sm.Xs[ixj];
          const bool up = ((tid & k2) == 0);
          if ((a > b) == up) { sm.Xs[tid] = b; sm.Xs[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    // O-W1 statistics
    const double h = __dmul_rn(0.95, (double)(kG - 1));
    const int f = (int)floor(h);
    const double frac = __dsub_rn(h, (double)f);
    const double q95 = (f + 1 < kG) ? __dadd_rn(sm.Xs[f], __dmul_rn(frac, __dsub_rn(sm.Xs[f + 1], sm.Xs[f]))) : sm.Xs[f];
    const double mn = sm.Xs[0], mx = sm.Xs[kG - 1];
    double sum = 0.0;
    for (int e = 0; e < kG; ++e) sum = __dadd_rn(sum, sm.X[e]);
    const double mean = __ddiv_rn(sum, (double)kG);
    // O-W2 candidate-set parameters (Eq. 8-11)
    const double s_min = __dmul_rn(p.s_min_factor, q95);
    double s_max = __dmul_rn(1.1, __dsub_rn(mx, mn));
    if (s_max <= s_min) s_max = __dmul_rn(1.01, s_min);
    const double s_gran = __ddiv_rn(__dsub_rn(s_max, s_min), (double)p.n_scale);
    const double b_max = __ddiv_rn(__dmul_rn(2.0, fabs(mean)), (double)K);
    const double b_min = -b_max;
    const double b_gran = __ddiv_rn(__dsub_rn(b_max, b_min), (double)p.n_bias);
    s_scal[0] = s_min; s_scal[1] = s_gran; s_scal[2] = b_min; s_scal[3] = b_gran;
  }
  __syncthreads();
  for (int j = tid; j < p.n_scale; j += blockDim.x)
    sm.S[j] = f16_bits_to_f64(f64_to_f16_bits(__dadd_rn(s_scal[0], __dmul_rn((double)(j + 1), s_scal[1]))));
  for (int k = tid; k < p.n_bias; k += blockDim.x)
    sm.B[k] = f16_bits_to_f64(f64_to_f16_bits(__dadd_rn(s_scal[2], __dmul_rn((double)k, s_scal[3]))));
  __syncthreads();
}

// MSE of the group under c_t = s r^t + b (Eq. 4): 2^K subset sums, nearest per element, SSE in element
// order, /128 -- every op an explicit _rn intrinsic (bit-identical to the oracle's evaluation).
template <int K>
__device__ __forceinline__ double entry_mse(const double* X, double r, double s, double b) {
  constexpr int NPTS = 1 << K;
  double c[K];
  double pw = 1.0;
#pragma unroll
  for (int t = 0; t < K; ++t) {
    c[t] = __dadd_rn(__dmul_rn(s, pw), b);
    pw = __dmul_rn(pw, r);
  }
  double v[NPTS];
#pragma unroll
  for (int m = 0; m < NPTS; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t)
      if ((m >> t) & 1) acc = __dadd_rn(acc, c[t]);
    v[m] = acc;
  }
  double sse = 0.0;
#pragma unroll 2
  for (int el = 0; el < kG; ++el) {
    const double x = X[el];
    double d = fabs(__dsub_rn(x, v[0]));
#pragma unroll
    for (int m = 1; m < NPTS; ++m) d = fmin(d, fabs(__dsub_rn(x, v[m])));
    sse = __dadd_rn(sse, __dmul_rn(d, d));
  }
  return __ddiv_rn(sse, (double)kG);
}

// Algorithm 1: entries strided over threads (R outer, S middle, B inner); a CTA arg-min on
// (mse, entry index) equals the sequential strict '<' scan.  Result in *win_e, *win_mse.
template <int K>
__device__ void grp_search(const EncParams& p, const GroupSmem& sm, double* red_mse, int* red_e, int* win_e,
                           double* win_mse) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = p.n_ratio * p.n_scale * p.n_bias, SB = p.n_scale * p.n_bias;
  double best = DBL_MAX;
  int best_e = 0x7fffffff;
  bool have = false;
  for (int e = tid; e < E; e += blockDim.x) {
    const int i = e / SB, rem = e - i * SB, j = rem / p.n_bias, k = rem - j * p.n_bias;
    const double mse = entry_mse<K>(sm.X, sm.R[i], sm.S[j], sm.B[k]);
    if (!have || mse < best) { best = mse; best_e = e; have = true; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, best, o);
    const int oe = __shfl_xor_sync(0xffffffffu, best_e, o);
    if (om < best || (om == best && oe < best_e)) { best = om; best_e = oe; }
  }
  if (lane == 0) { red_mse[warp] = best; red_e[warp] = best_e; }
  __syncthreads();
  if (tid == 0) {
    double bm = red_mse[0];
    int be = red_e[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (red_mse[w] < bm || (red_mse[w] == bm && red_e[w] < be)) { bm = red_mse[w]; be = red_e[w]; }
    *win_e = be;
    *win_mse = bm;
  }
  __syncthreads();
}

// Fast mode (sbvr_encode_config.strict = 0): the same MSE in fp32 (same formula, fp32 rounding).
template <int K>
__device__ __forceinline__ float entry_mse32(const double* X, float r, float s, float b) {
  constexpr int NPTS = 1 << K;
  float c[K];
  float pw = 1.f;
#pragma unroll
  for (int t = 0; t < K; ++t) {
    c[t] = fmaf(s, pw, b);
    pw *= r;
  }
  float v[NPTS];
#pragma unroll
  for (int m = 0; m < NPTS; ++m) {
    float acc = 0.f;
#pragma unroll
    for (int t = 0; t < K; ++t)
      if ((m >> t) & 1) acc += c[t];
    v[m] = acc;
  }
  float sse = 0.f;
#pragma unroll 4
  for (int el = 0; el < kG; ++el) {
    const float x = (float)X[el];
    float d = fabsf(x - v[0]);
#pragma unroll
    for (int m = 1; m < NPTS; ++m) d = fminf(d, fabsf(x - v[m]));
    sse = fmaf(d, d, sse);
  }
  return sse * (1.0f / kG);
}

// Fast-mode Algorithm 1: pass 1 evaluates every entry in fp32 (kept in shared memory when the space fits);
// pass 2 re-evaluates, with the strict fp64 entry_mse, every entry whose fp32 MSE is within a margin of the fp32
// best (the margin covers the fp32 error of a 128-term SSE many times over), and takes the strict arg-min of those
// in entry order.  Whenever the strict winner is in that set -- the margin makes that the rule -- the result is
// bit-identical to strict mode; the §8c.5 contract (strict MSE of the choice <= (1 + 1e-6) x the strict best) holds
// regardless of ties at the margin.
template <int K>
__device__ void grp_search_fast(const EncParams& p, const GroupSmem& sm, float* m32, int m32_cap, double* red_mse,
                                int* red_e, int* win_e, double* win_mse) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = p.n_ratio * p.n_scale * p.n_bias, SB = p.n_scale * p.n_bias;
  const bool keep = E <= m32_cap;
  float best32 = FLT_MAX, x2max = 0.f;
  for (int el = lane; el < kG; el += 32) x2max = fmaxf(x2max, (float)(sm.X[el] * sm.X[el]));
  for (int e = tid; e < E; e += blockDim.x) {
    const int i = e / SB, rem = e - i * SB, j = rem / p.n_bias, k = rem - j * p.n_bias;
    const float m = entry_mse32<K>(sm.X, (float)sm.R[i], (float)sm.S[j], (float)sm.B[k]);
    if (keep) m32[e] = m;
    best32 = fminf(best32, m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    best32 = fminf(best32, __shfl_xor_sync(0xffffffffu, best32, o));
    x2max = fmaxf(x2max, __shfl_xor_sync(0xffffffffu, x2max, o));
  }
  float* red32 = reinterpret_cast<float*>(red_mse);
  __syncthreads();
  if (lane == 0) red32[warp] = best32;
  __syncthreads();
  float b32 = red32[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b32 = fminf(b32, red32[w]);
  const float thr = b32 * (1.f + 1.f / 1024.f) + x2max * (1.f / (1 << 20));
  __syncthreads();
  double best = DBL_MAX;
  int best_e = 0x7fffffff;
  for (int e = tid; e < E; e += blockDim.x) {
    const int i = e / SB, rem = e - i * SB, j = rem / p.n_bias, k = rem - j * p.n_bias;
    const float m = keep ? m32[e] : entry_mse32<K>(sm.X, (float)sm.R[i], (float)sm.S[j], (float)sm.B[k]);
    if (m <= thr) {
      const double mse = entry_mse<K>(sm.X, sm.R[i], sm.S[j], sm.B[k]);
      if (mse < best) { best = mse; best_e = e; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, best, o);
    const int oe = __shfl_xor_sync(0xffffffffu, best_e, o);
    if (om < best || (om == best && oe < best_e)) { best = om; best_e = oe; }
  }
  if (lane == 0) { red_mse[warp] = best; red_e[warp] = best_e; }
  __syncthreads();
  if (tid == 0) {
    double bm = red_mse[0];
    int be = red_e[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (red_mse[w] < bm || (red_mse[w] == bm && red_e[w] < be)) { bm = red_mse[w]; be = red_e[w]; }
    *win_e = be;
    *win_mse = bm;
  }
  __syncthreads();
}

// P:231 bit assignment for coefficients (r, s, b) and the stores of planes / meta / mse.
template <int K>
__device__ void grp_assign_store(const EncParams& p, const GroupSmem& sm, int row, int g, double r, double s, double b,
                                 int ri, double mse, int hit) {
  constexpr int NPTS = 1 << K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Layout Lo(p.M, p.N, K);
  if (tid < kG) {
    double c[K];
    double pw = 1.0;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      c[t] = __dadd_rn(__dmul_rn(s, pw), b);
      pw = __dmul_rn(pw, r);
    }
    const double x = sm.X[tid];
    int bm = 0;
    double bd = 0.0, bv = 0.0;
#pragma unroll
    for (int m = 0; m < NPTS; ++m) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < K; ++t)
        if ((m >> t) & 1) acc = __dadd_rn(acc, c[t]);
      const double d = fabs(__dsub_rn(x, acc));
      if (m == 0 || d < bd || (d == bd && acc < bv)) { bd = d; bv = acc; bm = m; }
    }
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const uint32_t word = __ballot_sync(0xffffffffu, (bm >> t) & 1);
      if (lane == t) *reinterpret_cast<uint32_t*>(p.data + Lo.plane_byte(row, g, t, warp)) = word;
    }
  }
  if (tid == 0) {
    const long q = (long)row * Lo.NG + g;
    *reinterpret_cast<uint32_t*>(p.data + Lo.sb_byte(row, g)) =
        (uint32_t)f64_to_f16_bits(s) | ((uint32_t)f64_to_f16_bits(b) << 16);
    p.data[Lo.ri_byte(row, g)] = (uint8_t)ri;
    if (p.group_mse) p.group_mse[q] = mse;
    if (p.group_hit) p.group_hit[q] = (uint8_t)hit;
  }
  __syncthreads();
}

template <int K>
__global__ void __launch_bounds__(256) encode_weights_kernel(EncParams p) {
  extern __shared__ double smem[];
  GroupSmem sm;
  sm.X = smem;
  sm.Xs = sm.X + kG;
  sm.R = sm.Xs + kG;
  sm.S = sm.R + 64;
  sm.B = sm.S + p.n_scale;
  // fast mode: the fp32 MSE of every entry, after the candidate sets (m32_cap entries; 0 in strict mode)
  float* m32 = reinterpret_cast<float*>(sm.B + p.n_bias);
  const int m32_cap = p.fast ? p.m32_cap : 0;
  __shared__ double s_scal[4];       // s_min, s_gran, b_min, b_gran
  __shared__ double red_mse[8];
  __shared__ int red_e[8];
  __shared__ int win_e;
  __shared__ double win_mse;

  const int tid = threadIdx.x;
  const Layout Lo(p.M, p.N, K);
  const long n_groups = (long)p.M * Lo.NG;
  const int SB = p.n_scale * p.n_bias;
  for (int i = tid; i < p.n_ratio; i += blockDim.x) sm.R[i] = ratio_value(i, p.n_ratio);

  for (long q = blockIdx.x; q < n_groups; q += gridDim.x) {
    const int row = (int)(q / Lo.NG), g = (int)(q % Lo.NG);
    grp_load(p, sm, row, g);
    grp_candidates<K>(p, sm, s_scal);
    if (p.fast)
      grp_search_fast<K>(p, sm, m32, m32_cap, red_mse, red_e, &win_e, &win_mse);
    else
      grp_search<K>(p, sm, red_mse, red_e, &win_e, &win_mse);
    const int we = win_e;
    const int wi = we / SB, wrem = we - wi * SB, wj = wrem / p.n_bias, wk = wrem - wj * p.n_bias;
    grp_assign_store<K>(p, sm, row, g, sm.R[wi], sm.S[wj], sm.B[wk], wi, win_mse, 0);
  }
}

// Encode-time coefficient cache (P:233 and its footnote; reading A22): one CTA per row, groups left to
// right; an MRU cache of up to cache_size (r index, s, b) triples; the best cached entry (strict '<' in
// MRU order) is taken when its MSE is strictly below the moving average of accepted MSEs (initialised to
// the row's first full-search MSE, ema = (1-alpha) ema + alpha mse); otherwise Algorithm 1 runs and its
// winner goes to the front (an identical triple is moved, the least recent entry falls out).
template <int K>
__global__ void __launch_bounds__(256) encode_weights_cached_kernel(EncParams p) {
  extern __shared__ double smem[];
  GroupSmem sm;
  sm.X = smem;
  sm.Xs = sm.X + kG;
  sm.R = sm.Xs + kG;
  sm.S = sm.R + 64;
  sm.B = sm.S + p.n_scale;
  __shared__ double s_scal[4];
  __shared__ double red_mse[8];
  __shared__ int red_e[8];
  __shared__ int win_e;
  __shared__ double win_mse;
  __shared__ int c_ri[64];
  __shared__ double c_s[64], c_b[64], c_mse[64];
  __shared__ int n_c, have_ema, hit, bidx;
  __shared__ double ema;

  const int tid = threadIdx.x;
  const Layout Lo(p.M, p.N, K);
  const int SB = p.n_scale * p.n_bias;
  for (int i = tid; i < p.n_ratio; i += blockDim.x) sm.R[i] = ratio_value(i, p.n_ratio);
  for (int row = blockIdx.x; row < p.M; row += gridDim.x) {
    if (tid == 0) { n_c = 0; have_ema = 0; ema = 0.0; }
    __syncthreads();
    for (int g = 0; g < Lo.NG; ++g) {
      grp_load(p, sm, row, g);
      __syncthreads();
      const int nc = n_c;
      if (nc > 0 && have_ema && tid < nc) c_mse[tid] = entry_mse<K>(sm.X, sm.R[c_ri[tid]], c_s[tid], c_b[tid]);
      __syncthreads();
      if (tid == 0) {
        int h = 0, bi = -1;
        if (nc > 0 && have_ema) {
          double best = DBL_MAX;
          for (int k = 0; k < nc; ++k)
            if (bi < 0 || c_mse[k] < best) { best = c_mse[k]; bi = k; }
          h = best < ema;
        }
        hit = h;
        bidx = bi;
      }
      __syncthreads();
      int ri;
      double sv, bv, m;
      if (hit) {
        ri = c_ri[bidx]; sv = c_s[bidx]; bv = c_b[bidx]; m = c_mse[bidx];
      } else {
        grp_candidates<K>(p, sm, s_scal);
        grp_search<K>(p, sm, red_mse, red_e, &win_e, &win_mse);
        const int we = win_e;
        const int wi = we / SB, wrem = we - wi * SB, wj = wrem / p.n_bias, wk = wrem - wj * p.n_bias;
        ri = wi; sv = sm.S[wj]; bv = sm.B[wk]; m = win_mse;
      }
      __syncthreads();
      if (tid == 0) {
        int at;
        if (hit) {
          at = bidx;
        } else {
          at = -1;
          for (int k = 0; k < n_c; ++k)
            if (c_ri[k] == ri && c_s[k] == sv && c_b[k] == bv) { at = k; break; }
          if (at < 0) {
            if (n_c < p.cache_size) ++n_c;
            at = n_c - 1;
          }
        }
        for (int k = at; k > 0; --k) { c_ri[k] = c_ri[k - 1]; c_s[k] = c_s[k - 1]; c_b[k] = c_b[k - 1]; }
        if (p.cache_size > 0) { c_ri[0] = ri; c_s[0] = sv; c_b[0] = bv; }
        if (!have_ema) { ema = m; have_ema = 1; }
        else ema = __dadd_rn(__dmul_rn(__dsub_rn(1.0, p.cache_alpha), ema), __dmul_rn(p.cache_alpha, m));
      }
      const int hh = hit;
      grp_assign_store<K>(p, sm, row, g, sm.R[ri], sv, bv, ri, m, hh);
    }
  }
}

// ---------------------------------------------------------------- f2: coefficient table + per-group index
// (reading A23).  Step 1: Algorithm 1 on the evenly spaced sample groups; their winners are
// written to cand[2i] = s16 | b16 << 16, cand[2i + 1] = r index.
template <int K>
__global__ void __launch_bounds__(256) encode_sample_kernel(EncParams p, int n_sample, uint32_t* cand) {
  extern __shared__ double smem[];
  GroupSmem sm;
  sm.X = smem;
  sm.Xs = sm.X + kG;
  sm.R = sm.Xs + kG;
  sm.S = sm.R + 64;
  sm.B = sm.S + p.n_scale;
  __shared__ double s_scal[4];
  __shared__ double red_mse[8];
  __shared__ int red_e[8];
  __shared__ int win_e;
  __shared__ double win_mse;
  const int tid = threadIdx.x;
  const int NG = p.N / kG;
  const long n_groups = (long)p.M * NG;
  const int SB = p.n_scale * p.n_bias;
  for (int i = tid; i < p.n_ratio; i += blockDim.x) sm.R[i] = ratio_value(i, p.n_ratio);
  for (int i = blockIdx.x; i < n_sample; i += gridDim.x) {
    const long q = (long)i * n_groups / n_sample;
    const int row = (int)(q / NG), g = (int)(q % NG);
    grp_load(p, sm, row, g);
    grp_candidates<K>(p, sm, s_scal);
    grp_search<K>(p, sm, red_mse, red_e, &win_e, &win_mse);
    if (tid == 0) {
      const int we = win_e;
      const int wi = we / SB, wrem = we - wi * SB, wj = wrem / p.n_bias, wk = wrem - wj * p.n_bias;
      cand[2 * i] = (uint32_t)f64_to_f16_bits(sm.S[wj]) | ((uint32_t)f64_to_f16_bits(sm.B[wk]) << 16);
      cand[2 * i + 1] = (uint32_t)wi;
    }
    __syncthreads();
  }
}

// Step 2: the table = distinct sample winners in sample order (word 0 = entry count).
__global__ void table_dedupe_kernel(const uint32_t* cand, int n_sample, uint32_t* table) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int n = 0;
  for (int i = 0; i < n_sample; ++i) {
    const uint32_t a = cand[2 * i], b = cand[2 * i + 1];
    bool dup = false;
    for (int j = 0; j < n && !dup; ++j) dup = table[1 + 2 * j] == a && table[2 + 2 * j] == b;
    if (!dup) {
      table[1 + 2 * n] = a;
      table[2 + 2 * n] = b;
      ++n;
    }
  }
  table[0] = (uint32_t)n;
}

// Step 3: every group takes the table entry of least MSE (strict '<' in table order = a CTA arg-min on
// (mse, entry)); its bits are assigned for that entry and stored in the indexed layout.
template <int K>
__global__ void __launch_bounds__(256) encode_indexed_kernel(EncParams p, const uint32_t* table) {
  constexpr int NPTS = 1 << K;
  __shared__ double X[kG];
  __shared__ double R[64];
  __shared__ double red_mse[8];
  __shared__ int red_e[8];
  __shared__ int win_e;
  __shared__ double win_mse;
  __shared__ uint32_t s_tab[2 * kMaxTable];
  __shared__ int s_n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const IdxLayout Lo(p.M, p.N, K);
  const long n_groups = (long)p.M * Lo.NG;
  for (int i = tid; i < p.n_ratio; i += blockDim.x) R[i] = ratio_value(i, p.n_ratio);
  if (tid == 0) s_n = (int)table[0];
  __syncthreads();
  for (int i = tid; i < 2 * s_n; i += blockDim.x) s_tab[i] = table[1 + i];
  __syncthreads();
  const int n = s_n;
  for (long q = blockIdx.x; q < n_groups; q += gridDim.x) {
    const int row = (int)(q / Lo.NG), g = (int)(q % Lo.NG);
    if (tid < kG) X[tid] = load_w(p.W, p.dtype, (size_t)row * p.N + (size_t)g * kG + tid);
    __syncthreads();
    double best = DBL_MAX;
    int best_e = 0x7fffffff;
    for (int e = tid; e < n; e += blockDim.x) {
      const uint32_t sb = s_tab[2 * e];
      const double m = entry_mse<K>(X, R[s_tab[2 * e + 1]], f16_bits_to_f64((uint16_t)(sb & 0xffffu)),
                                    f16_bits_to_f64((uint16_t)(sb >> 16)));
      if (m < best || (m == best && e < best_e)) { best = m; best_e = e; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(0xffffffffu, best, o);
      const int oe = __shfl_xor_sync(0xffffffffu, best_e, o);
      if (om < best || (om == best && oe < best_e)) { best = om; best_e = oe; }
    }
    if (lane == 0) { red_mse[warp] = best; red_e[warp] = best_e; }
    __syncthreads();
    if (tid == 0) {
      double bm = red_mse[0];
      int be = red_e[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (red_mse[w] < bm || (red_mse[w] == bm && red_e[w] < be)) { bm = red_mse[w]; be = red_e[w]; }
      win_e = be;
      win_mse = bm;
    }
    __syncthreads();
    const int we = win_e;
    const uint32_t sb = s_tab[2 * we];
    const double r = R[s_tab[2 * we + 1]], s = f16_bits_to_f64((uint16_t)(sb & 0xffffu)),
                 b = f16_bits_to_f64((uint16_t)(sb >> 16));
    if (tid < kG) {
      double c[K];
      double pw = 1.0;
#pragma unroll
      for (int t = 0; t < K; ++t) {
        c[t] = __dadd_rn(__dmul_rn(s, pw), b);
        pw = __dmul_rn(pw, r);
      }
      const double x = X[tid];
      int bm = 0;
      double bd = 0.0, bv = 0.0;
#pragma unroll
      for (int m = 0; m < NPTS; ++m) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < K; ++t)
          if ((m >> t) & 1) acc = __dadd_rn(acc, c[t]);
        const double d = fabs(__dsub_rn(x, acc));
        if (m == 0 || d < bd || (d == bd && acc < bv)) { bd = d; bv = acc; bm = m; }
      }
#pragma unroll
      for (int t = 0; t < K; ++t) {
        const uint32_t word = __ballot_sync(0xffffffffu, (bm >> t) & 1);
        if (lane == t) *reinterpret_cast<uint32_t*>(p.data + Lo.plane_byte(row, g, t, warp)) = word;
      }
    }
    if (tid == 0) {
      p.data[Lo.idx_byte(row, g)] = (uint8_t)we;
      if (p.group_mse) p.group_mse[(long)row * Lo.NG + g] = win_mse;
    }
    __syncthreads();
  }
}

__global__ void ratio_table_kernel(float* out, int n_ratio, int K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_ratio) return;
  const double r = ratio_value(i, n_ratio);
  double pw = 1.0;
  for (int t = 0; t < K; ++t) {
    out[i * K + t] = __double2float_rn(pw);
    pw = __dmul_rn(pw, r);
  }
}

sbvr_status launch_ratio_table(float* ratio_pow, int n_ratio, int K, cudaStream_t st) {
  ratio_table_kernel<<<1, 64, 0, st>>>(ratio_pow, n_ratio, K);
  return check_launch("ratio_table_kernel");
}

template <int K>
static sbvr_status launch_k(const EncParams& p_in, bool cached, cudaStream_t st) {
  EncParams p = p_in;
  const long E = (long)p.n_ratio * p.n_scale * p.n_bias;
  p.m32_cap = (p.fast && !cached) ? (int)(E <= 32768 ? E : 0) : 0;   // <= 128 KB of fp32 MSEs, else recomputed
  const size_t smem = sizeof(double) * (2 * kG + 64 + p.n_scale + p.n_bias) + sizeof(float) * p.m32_cap;
  if (smem > 48 * 1024 - 2048) {
    cudaError_t e = cudaFuncSetAttribute(encode_weights_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(encode_weights_cached_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(e));
  }
  if (cached) {
    const int grid = p.M < (1 << 30) ? p.M : (1 << 30);
    encode_weights_cached_kernel<K><<<grid, 256, smem, st>>>(p);
    return check_launch("encode_weights_cached_kernel");
  }
  const long groups = (long)p.M * (p.N / kG);
  const int grid = (int)(groups < (1L << 30) ? groups : (1L << 30));
  encode_weights_kernel<K><<<grid, 256, smem, st>>>(p);
  return check_launch("encode_weights_kernel");
}

sbvr_status launch_encode_weights(const sbvr_encode_config* cfg, const void* W, int dtype, int M, int N,
                                  const sbvr_weights* out, double* group_mse, int cache_size, double cache_alpha,
                                  uint8_t* group_hit, cudaStream_t st) {
  EncParams p;
  p.cache_size = cache_size;
  p.cache_alpha = cache_alpha;
  p.group_hit = group_hit;
  const bool cached = cache_size >= 0;
  p.W = W; p.dtype = dtype; p.M = M; p.N = N;
  p.n_ratio = cfg->n_ratio; p.n_scale = cfg->n_scale; p.n_bias = cfg->n_bias;
  p.s_min_factor = cfg->s_min_factor;
  p.data = out->data;
  p.group_mse = group_mse;
  p.fast = cfg->strict ? 0 : 1;
  p.m32_cap = 0;
  sbvr_status s;
  switch (cfg->K) {
    case 1: s = launch_k<1>(p, cached, st); break;
    case 2: s = launch_k<2>(p, cached, st); break;
    case 3: s = launch_k<3>(p, cached, st); break;
    case 4: s = launch_k<4>(p, cached, st); break;
    case 5: s = launch_k<5>(p, cached, st); break;
    case 6: s = launch_k<6>(p, cached, st); break;
    default: return set_error(SBVR_ERR_UNSUPPORTED, "encoder K=%d", cfg->K);
  }
  if (s != SBVR_OK) return s;
  return launch_ratio_table(out->ratio_pow, cfg->n_ratio, cfg->K, st);
}

template <int K>
static sbvr_status launch_indexed_k(const EncParams& p, int n_sample, uint32_t* cand, uint32_t* table, cudaStream_t st) {
  const size_t smem = sizeof(double) * (2 * kG + 64 + p.n_scale + p.n_bias);
  if (smem > 48 * 1024 - 2048) {
    cudaError_t e = cudaFuncSetAttribute(encode_sample_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(SBVR_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(e));
  }
  encode_sample_kernel<K><<<n_sample, 256, smem, st>>>(p, n_sample, cand);
  sbvr_status s = check_launch("encode_sample_kernel");
  if (s != SBVR_OK) return s;
  table_dedupe_kernel<<<1, 32, 0, st>>>(cand, n_sample, table);
  s = check_launch("table_dedupe_kernel");
  if (s != SBVR_OK) return s;
  const long groups = (long)p.M * (p.N / kG);
  const int grid = (int)(groups < (1L << 30) ? groups : (1L << 30));
  encode_indexed_kernel<K><<<grid, 256, 0, st>>>(p, table);
  return check_launch("encode_indexed_kernel");
}

sbvr_status launch_encode_indexed(const sbvr_encode_config* cfg, int n_table, const void* W, int dtype, int M, int N,
                                  const sbvr_weights* out, double* group_mse, uint32_t* cand, cudaStream_t st) {
  EncParams p = {};
  p.W = W; p.dtype = dtype; p.M = M; p.N = N;
  p.n_ratio = cfg->n_ratio; p.n_scale = cfg->n_scale; p.n_bias = cfg->n_bias;
  p.s_min_factor = cfg->s_min_factor;
  p.data = out->data;
  p.group_mse = group_mse;
  p.cache_size = -1;
  const long groups = (long)M * (N / kG);
  const int n_sample = (int)(n_table < groups ? n_table : groups);
  sbvr_status s;
  switch (cfg->K) {
    case 1: s = launch_indexed_k<1>(p, n_sample, cand, out->coef_table, st); break;
    case 2: s = launch_indexed_k<2>(p, n_sample, cand, out->coef_table, st); break;
    case 3: s = launch_indexed_k<3>(p, n_sample, cand, out->coef_table, st); break;
    case 4: s = launch_indexed_k<4>(p, n_sample, cand, out->coef_table, st); break;
    case 5: s = launch_indexed_k<5>(p, n_sample, cand, out->coef_table, st); break;
    case 6: s = launch_indexed_k<6>(p, n_sample, cand, out->coef_table, st); break;
    default: return set_error(SBVR_ERR_UNSUPPORTED, "encoder K=%d", cfg->K);
  }
  if (s != SBVR_OK) return s;
  return launch_ratio_table(out->ratio_pow, cfg->n_ratio, cfg->K, st);
}

}  // namespace sbvr
