/*
 * sbvr_oracle.c -- CPU ORACLE for SBVR (arXiv 2509.18172).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2509_18172_b200/) never does,
 * and this file shares no code, headers, tables or constant generators with it.
 *
 * Plain, slow, obviously-correct fp64 C, compiled with -ffp-contract=off so that every
 * `a*b+c` below is two IEEE roundings, in the order written.  Each function cites the
 * passage of /root/reference/PAPER.md ("P:<line>") it restates; where the paper is
 * silent or garbled the reading used is the one listed in DESIGN.md §Readings (A1..A20,
 * numbering from SURVEY.md §8c.3).
 *
 * Canonical interchange layouts (plain conventions, no arithmetic):
 *   weight planes : [M][N/G][K][G/32] uint32, LSB-first (bit i of word w = element 32w+i)
 *   weight meta   : s16, b16 [M][N/G] fp16 bit patterns; r_idx [M][N/G] uint8
 *   activation    : z [N] int32; planes [N/G][l][G/32] uint32; scales [N/G] fp32
 *
 * Parity status: every exported function is pinned by tests/test_oracle_*.py against
 * brute force, closed forms, numpy library routines or worked examples; none is
 * "parity unpinned" (see DESIGN.md §Oracle pins).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAX_K 8
#define OR_MAX_PTS (1 << OR_MAX_K)
#define OR_MAX_G 1024

typedef struct {
  int32_t K;            /* number of coefficients / bit-planes */
  int32_t group_size;   /* elements per group, 128 typical */
  int32_t n_ratio;      /* |R| */
  int32_t n_scale;      /* |S| */
  int32_t n_bias;       /* |B| */
  double s_min_factor;  /* s_min = s_min_factor * q95(D); 2.0 is the paper (reading A1) */
} oracle_cfg;

/* ---------------------------------------------------------------- fp16 storage rounding
 * Reading A15: the scale and bias candidates are rounded to the storage dtype (IEEE
 * binary16, round-to-nearest-even) before the search.  Written out from the binary16
 * definition: 1 sign bit, 5 exponent bits (bias 15), 10 fraction bits; subnormals below
 * 2^-14 with quantum 2^-24; overflow to infinity.                                        */
uint16_t oracle_fp16_bits(double x) {
  uint16_t sign = 0;
  if (x != x) return 0x7e00;               /* NaN */
  if (x < 0 || (x == 0 && signbit(x))) { sign = 0x8000; x = -x; }
  if (x == 0) return sign;
  if (isinf(x)) return sign | 0x7c00;
  int e;
  double m = frexp(x, &e);                 /* x = m * 2^e, m in [0.5, 1) exactly */
  int E = e - 1;                           /* x = (2m) * 2^E, 2m in [1, 2) */
  double q;                                /* quantum at this binade */
  if (E < -14) q = ldexp(1.0, -24);        /* subnormal range */
  else q = ldexp(1.0, E - 10);
  double k = x / q;                        /* exact: power-of-two division */
  double kf = floor(k);
  double rem = k - kf;                     /* exact */
  if (rem > 0.5 || (rem == 0.5 && fmod(kf, 2.0) != 0.0)) kf += 1.0;
  double r = kf * q;                       /* exact */
  if (r >= 65520.0 || r > 65504.0) return sign | 0x7c00;   /* overflow to inf */
  /* encode r (now exactly representable) */
  if (r < ldexp(1.0, -14)) {
    return sign | (uint16_t)(r / ldexp(1.0, -24));
  }
  int e2;
  double m2 = frexp(r, &e2);
  int E2 = e2 - 1;
  uint16_t frac = (uint16_t)((2.0 * m2 - 1.0) * 1024.0);
  return sign | (uint16_t)((E2 + 15) << 10) | frac;
}

double oracle_fp16_to_double(uint16_t h) {
  int sign = (h >> 15) & 1, exp = (h >> 10) & 0x1f, frac = h & 0x3ff;
  double v;
  if (exp == 0) v = ldexp((double)frac, -24);
  else if (exp == 31) v = frac ? NAN : INFINITY;
  else v = ldexp(1.0 + frac / 1024.0, exp - 15);
  return sign ? -v : v;
}

/* ---------------------------------------------------------------- O-W1 statistics
 * P:187 s_min = 2 q95(D); "q95(D) denotes the 95th percentile"; P:186 avg(D);
 * P:185 max(D), min(D).  Reading A6: linear interpolation on the sorted data with
 * h = 0.95 (n-1); q95 = D[floor h] + (h - floor h) (D[floor h + 1] - D[floor h]).
 * The mean is the left-to-right sum in element order divided by n.                    */
static int cmp_dbl(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

void oracle_group_stats(const double* D, int n, double* q95, double* dmin, double* dmax, double* mean) {
  double sorted[OR_MAX_G];
  memcpy(sorted, D, sizeof(double) * (size_t)n);
  qsort(sorted, (size_t)n, sizeof(double), cmp_dbl);
  double h = 0.95 * (double)(n - 1);
  int f = (int)floor(h);
  double frac = h - (double)f;
  if (f + 1 < n) *q95 = sorted[f] + frac * (sorted[f + 1] - sorted[f]);
  else *q95 = sorted[f];
  *dmin = sorted[0];
  *dmax = sorted[n - 1];
  double sum = 0.0;
  for (int e = 0; e < n; ++e) sum = sum + D[e];
  *mean = sum / (double)n;
}

/* ---------------------------------------------------------------- O-W2 candidate sets
 * Eq. 5-11, taken literally (readings A1, A2, A3, A7):
 *   S = { s_min + (j+1) s_gran | 0 <= j < N_scale }        (Eq. 6)
 *   B = { b_min + k b_gran     | 0 <= k < N_bias }         (Eq. 7)
 *   s_max = 1.1 (max D - min D)                            (Eq. 8)
 *   b_max = 2 |avg D| / K, b_min = -b_max                  (Eq. 9, 10)
 *   s_min = 2 q95(D)                                       (Eq. 10)
 *   s_gran = (s_max - s_min)/N_scale, b_gran = (b_max - b_min)/N_bias   (Eq. 11)
 * Degenerate guard (reading A18): if s_max <= s_min then s_max = 1.01 s_min.
 * R (reading A3): two disjoint sets of N_ratio/2 points, numpy-linspace spaced
 * over [-1, -0.5] then [0.5, 1], endpoints inclusive.
 * S and B are rounded to fp16 (reading A15) and used as the rounded fp64 values.      */
void oracle_ratio_set(int n_ratio, double* R) {
  int half = n_ratio / 2;
  for (int part = 0; part < 2; ++part) {
    double a = part == 0 ? -1.0 : 0.5;
    double b = part == 0 ? -0.5 : 1.0;
    for (int i = 0; i < half; ++i) {
      double v;
      if (half == 1) v = a;
      else if (i == half - 1) v = b;
      else v = (double)i * ((b - a) / (double)(half - 1)) + a;
      R[part * half + i] = v;
    }
  }
}

void oracle_candidates(const double* D, int n, const oracle_cfg* cfg, double* R, double* S, double* B) {
  double q95, mn, mx, mean;
  oracle_group_stats(D, n, &q95, &mn, &mx, &mean);
  double s_min = cfg->s_min_factor * q95;
  double s_max = 1.1 * (mx - mn);
  if (s_max <= s_min) s_max = 1.01 * s_min;
  double s_gran = (s_max - s_min) / (double)cfg->n_scale;
  for (int j = 0; j < cfg->n_scale; ++j) {
    double s = s_min + (double)(j + 1) * s_gran;
    S[j] = oracle_fp16_to_double(oracle_fp16_bits(s));
  }
  double b_max = (2.0 * fabs(mean)) / (double)cfg->K;
  double b_min = -b_max;
  double b_gran = (b_max - b_min) / (double)cfg->n_bias;
  for (int k = 0; k < cfg->n_bias; ++k) {
    double b = b_min + (double)k * b_gran;
    B[k] = oracle_fp16_to_double(oracle_fp16_bits(b));
  }
  oracle_ratio_set(cfg->n_ratio, R);
}

/* ---------------------------------------------------------------- O-W3 coefficients
 * Eq. 4: c_t = s r^t + b, t = 0..K-1.  r^t by repeated multiplication
 * (p_0 = 1, p_{t+1} = p_t r); c_t = s*p_t then + b (two roundings).                     */
void oracle_coefficients(double r, double s, double b, int K, double* c) {
  double p = 1.0;
  for (int t = 0; t < K; ++t) {
    double sp = s * p;
    c[t] = sp + b;
    p = p * r;
  }
}

/* ---------------------------------------------------------------- O-W4 subset sums
 * P:131 ("given a coefficient set [a,b,c], our representation points become
 * [0,a,b,c,a+b,a+c,b+c,a+b+c]"); Alg. 1 note (1) AllSubsetSums.
 * v(m) = sum of c_t over the set bits t of m, added in increasing t starting from 0.0.
 * Output sorted ascending by (v, m)  (insertion sort, stable on m).                     */
void oracle_subset_sums(const double* c, int K, double* v_sorted, int32_t* m_sorted) {
  int n = 1 << K;
  for (int m = 0; m < n; ++m) {
    double v = 0.0;
    for (int t = 0; t < K; ++t)
      if ((m >> t) & 1) v = v + c[t];
    /* insert (v, m) keeping (v, m) order; m increases so equal v stay in m order */
    int i = m;
    while (i > 0 && v_sorted[i - 1] > v) {
      v_sorted[i] = v_sorted[i - 1];
      m_sorted[i] = m_sorted[i - 1];
      --i;
    }
    v_sorted[i] = v;
    m_sorted[i] = m;
  }
}

/* ---------------------------------------------------------------- O-W5 nearest
 * Alg. 1 note (2): "Return the sum that is closest to x".  Reading A8: linear
 * scan, strict '<' on |x - v|, so a distance tie keeps the earlier (smaller v; for equal
 * v the smaller mask) point.  Returns the index into the sorted list.                   */
int oracle_nearest(const double* v_sorted, int n_pts, double x) {
  int best = 0;
  double bd = fabs(x - v_sorted[0]);
  for (int i = 1; i < n_pts; ++i) {
    double d = fabs(x - v_sorted[i]);
    if (d < bd) { bd = d; best = i; }
  }
  return best;
}

/* ---------------------------------------------------------------- O-W6 search (Algorithm 1)
 * Algorithm 1: input weight vector X and search space S = R x S x B (Eq. 4,
 * P:152-169); e* <- nil, bestMSE <- inf; for each entry e (order R outer, S middle,
 * B inner -- reading A8): sums <- AllSubsetSums(e); errorSum <- 0; for x in X (element
 * order): n <- Nearest(sums, x); errorSum <- errorSum + (x - n)^2; mse <- errorSum/|X|;
 * if mse < bestMSE (strict): e* <- e.  Returns bestMSE; writes the winning indices.     */
double oracle_search(const double* X, int n, int K, const double* R, int nR, const double* S, int nS,
                     const double* B, int nB, int32_t* bi_out, int32_t* bj_out, int32_t* bk_out) {
  const int npts = 1 << K;
  double best_mse = INFINITY;
  int bi = 0, bj = 0, bk = 0;
  double c[OR_MAX_K], v[OR_MAX_PTS];
  int32_t mk[OR_MAX_PTS];
  for (int i = 0; i < nR; ++i) {
    for (int j = 0; j < nS; ++j) {
      for (int k = 0; k < nB; ++k) {
        oracle_coefficients(R[i], S[j], B[k], K, c);
        oracle_subset_sums(c, K, v, mk);
        double error_sum = 0.0;
        for (int e = 0; e < n; ++e) {
          int idx = oracle_nearest(v, npts, X[e]);
          double d = X[e] - v[idx];
          error_sum = error_sum + d * d;
        }
        double mse = error_sum / (double)n;
        if (mse < best_mse) { best_mse = mse; bi = i; bj = j; bk = k; }
      }
    }
  }
  *bi_out = bi; *bj_out = bj; *bk_out = bk;
  return best_mse;
}

/* ---------------------------------------------------------------- O-W7 bit assignment
 * "For each element x_i in the weight vector, we identify the subset of elements
 * from the entry whose subset sum is closest to x_i.  We then mark the selected elements
 * as 1 and the others as 0" -- bit t of element e's mask goes to plane t (canonical
 * [K][n/32] LSB-first layout).                                                           */
void oracle_assign(const double* X, int n, const double* c, int K, uint32_t* planes) {
  const int npts = 1 << K;
  double v[OR_MAX_PTS];
  int32_t mk[OR_MAX_PTS];
  oracle_subset_sums(c, K, v, mk);
  memset(planes, 0, sizeof(uint32_t) * (size_t)K * (size_t)(n / 32));
  for (int e = 0; e < n; ++e) {
    int m = mk[oracle_nearest(v, npts, X[e])];
    for (int t = 0; t < K; ++t)
      if ((m >> t) & 1) planes[t * (n / 32) + e / 32] |= 1u << (e % 32);
  }
}

/* Encode one group: candidates (Eq. 5-11) -> search (Alg. 1) -> assignment.
 * Outputs planes [K][n/32], the stored fp16 s and b, r_idx and the entry index
 * ((i*n_scale)+j)*n_bias+k.  Returns the winning MSE.                                   */
double oracle_encode_group(const double* X, const oracle_cfg* cfg, uint32_t* planes, uint16_t* s16,
                           uint16_t* b16, uint8_t* r_idx, int32_t* entry_out) {
  const int n = cfg->group_size, K = cfg->K;
  double R[256], S[4096], B[4096];
  oracle_candidates(X, n, cfg, R, S, B);
  int32_t bi, bj, bk;
  double best = oracle_search(X, n, K, R, cfg->n_ratio, S, cfg->n_scale, B, cfg->n_bias, &bi, &bj, &bk);
  double c[OR_MAX_K];
  oracle_coefficients(R[bi], S[bj], B[bk], K, c);
  oracle_assign(X, n, c, K, planes);
  *s16 = oracle_fp16_bits(S[bj]);
  *b16 = oracle_fp16_bits(B[bk]);
  *r_idx = (uint8_t)bi;
  if (entry_out) *entry_out = (bi * cfg->n_scale + bj) * cfg->n_bias + bk;
  return best;
}

/* Encode a row-major M x N fp32 matrix, groups of G along N (reading A17).
 * Groups are independent ("grouping facilitates parallelism during the
 * encoding step"), so they are spread over OpenMP threads; each group's result does
 * not depend on the thread count.  Returns the number of threads used.                 */
int oracle_encode_matrix(const float* W, int M, int N, const oracle_cfg* cfg, uint32_t* planes, uint16_t* s16,
                         uint16_t* b16, uint8_t* r_idx, double* mse, int nthreads) {
  const int G = cfg->group_size, NG = N / G, K = cfg->K, WPG = G / 32;
  long total = (long)M * NG;
  int used = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
#pragma omp for schedule(dynamic, 4)
    for (long q = 0; q < total; ++q) {
#else
  (void)nthreads;
  {
    for (long q = 0; q < total; ++q) {
#endif
      long r = q / NG, g = q % NG;
      double X[OR_MAX_G];
      for (int e = 0; e < G; ++e) X[e] = (double)W[r * (long)N + g * G + e];
      double m = oracle_encode_group(X, cfg, planes + q * (long)K * WPG, s16 + q, b16 + q, r_idx + q, NULL);
      if (mse) mse[q] = m;
    }
  }
  return used;
}

/* ---------------------------------------------------------------- O-C encode-time coefficient cache
 * P:233 (§4.2 and its footnote): "we maintain a cache of previously selected variables r, s, and b.
 * The search algorithm first checks the cache to determine if any previously selected combinations
 * ... provide sufficient accuracy before exploring the entire search space" -- footnote: "We maintain a
 * moving average of the quantization error.  If the error from the cached values is below this moving
 * average, the cached values are used."  Reading A22: the cache is per row, groups are
 * visited left to right (a fixed order, so the result is deterministic and rows stay parallel); it holds
 * up to `cache_size` (r index, s, b) triples in most-recently-used order; the best cached entry (strict
 * '<' in MRU order) is used when its MSE is strictly below the moving average, which is initialised to
 * the row's first full-search MSE and updated with every accepted MSE as ema = (1-alpha) ema + alpha mse;
 * a hit moves the entry to the front, a miss runs Algorithm 1 and puts its winner in front (an identical
 * triple already cached is moved instead of duplicated; the least recent entry falls out when full).     */
double oracle_entry_mse(const double* X, int n, int K, double r, double s, double b) {
  const int npts = 1 << K;
  double c[OR_MAX_K], v[OR_MAX_PTS];
  int32_t mk[OR_MAX_PTS];
  oracle_coefficients(r, s, b, K, c);
  oracle_subset_sums(c, K, v, mk);
  double error_sum = 0.0;
  for (int e = 0; e < n; ++e) {
    double d = X[e] - v[oracle_nearest(v, npts, X[e])];
    error_sum = error_sum + d * d;
  }
  return error_sum / (double)n;
}

int oracle_encode_matrix_cached(const float* W, int M, int N, const oracle_cfg* cfg, int cache_size, double alpha,
                                uint32_t* planes, uint16_t* s16, uint16_t* b16, uint8_t* r_idx, double* mse,
                                uint8_t* hit_out) {
  const int G = cfg->group_size, NG = N / G, K = cfg->K, WPG = G / 32;
  double R[256];
  oracle_ratio_set(cfg->n_ratio, R);
  long hits = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : hits)
  for (long r = 0; r < M; ++r) {
    int c_ri[64];
    double c_s[64], c_b[64];
    int n_c = 0, have_ema = 0;
    double ema = 0.0;
    for (int g = 0; g < NG; ++g) {
      const long q = r * NG + g;
      double X[OR_MAX_G];
      for (int e = 0; e < G; ++e) X[e] = (double)W[r * (long)N + g * G + e];
      int hit = 0, bidx = -1;
      double best = INFINITY;
      if (n_c > 0 && have_ema) {
        for (int k = 0; k < n_c; ++k) {
          double m = oracle_entry_mse(X, G, K, R[c_ri[k]], c_s[k], c_b[k]);
          if (m < best) { best = m; bidx = k; }
        }
        if (best < ema) hit = 1;
      }
      int ri;
      double sv, bv, m;
      if (hit) {
        ri = c_ri[bidx]; sv = c_s[bidx]; bv = c_b[bidx]; m = best;
        for (int k = bidx; k > 0; --k) { c_ri[k] = c_ri[k - 1]; c_s[k] = c_s[k - 1]; c_b[k] = c_b[k - 1]; }
      } else {
        double Rr[256], S[4096], B[4096];
        oracle_candidates(X, G, cfg, Rr, S, B);
        int32_t bi, bj, bk;
        m = oracle_search(X, G, K, Rr, cfg->n_ratio, S, cfg->n_scale, B, cfg->n_bias, &bi, &bj, &bk);
        ri = bi; sv = S[bj]; bv = B[bk];
        int at = -1;
        for (int k = 0; k < n_c; ++k)
          if (c_ri[k] == ri && c_s[k] == sv && c_b[k] == bv) { at = k; break; }
        if (at < 0) {
          if (n_c < cache_size) ++n_c;
          at = n_c - 1;                      /* the least recent entry is overwritten when full */
        }
        for (int k = at; k > 0; --k) { c_ri[k] = c_ri[k - 1]; c_s[k] = c_s[k - 1]; c_b[k] = c_b[k - 1]; }
      }
      if (cache_size > 0) { c_ri[0] = ri; c_s[0] = sv; c_b[0] = bv; }
      if (!have_ema) { ema = m; have_ema = 1; }
      else ema = (1.0 - alpha) * ema + alpha * m;
      double c[OR_MAX_K];
      oracle_coefficients(R[ri], sv, bv, K, c);
      oracle_assign(X, G, c, K, planes + q * (long)K * WPG);
      s16[q] = oracle_fp16_bits(sv);
      b16[q] = oracle_fp16_bits(bv);
      r_idx[q] = (uint8_t)ri;
      if (mse) mse[q] = m;
      if (hit_out) hit_out[q] = (uint8_t)hit;
      hits += hit;
    }
  }
  return (int)hits;
}

/* ---------------------------------------------------------------- O-X activation conversion
 * §4.3 / Eq. 12: per vector (group of G, reading A12) scale
 * s_x = absmax / (2^(l-1) - 1) (reading A10), power-of-two coefficients
 * {-2^(l-1) s, s, 2s, ..., 2^(l-2) s} (reading A11: plane l-1 is the sign plane),
 * z = clamp(rne(x / s_x), -(2^(l-1)-1), 2^(l-1)-1); plane j bit e = bit j of z in
 * l-bit two's complement.  fp32 IEEE throughout (x is fp16, exactly representable).
 * All-zero group: s_x = 0, z = 0.                                          */
static float fp16_to_float(uint16_t h) { return (float)oracle_fp16_to_double(h); }

void oracle_encode_vector(const uint16_t* x16, int N, int G, int l, int32_t* z, uint32_t* planes, float* scales) {
  const int NG = N / G, WPG = G / 32;
  const int zmax = (1 << (l - 1)) - 1;
  memset(planes, 0, sizeof(uint32_t) * (size_t)NG * l * WPG);
  for (int g = 0; g < NG; ++g) {
    float absmax = 0.0f;
    for (int e = 0; e < G; ++e) {
      float a = fabsf(fp16_to_float(x16[g * G + e]));
      if (a > absmax) absmax = a;
    }
    float sx = 0.0f;
    if (absmax != 0.0f) sx = absmax / (float)zmax;
    scales[g] = sx;
    for (int e = 0; e < G; ++e) {
      int zi = 0;
      if (sx != 0.0f) {
        float q = fp16_to_float(x16[g * G + e]) / sx;
        float rq = rintf(q);             /* round-half-even in the default FP mode */
        zi = (int)rq;
        if (zi > zmax) zi = zmax;
        if (zi < -zmax) zi = -zmax;
      }
      z[g * G + e] = zi;
      uint32_t u = (uint32_t)zi & ((1u << l) - 1u);
      for (int j = 0; j < l; ++j)
        if ((u >> j) & 1u) planes[(g * l + j) * WPG + e / 32] |= 1u << (e % 32);
    }
  }
}

/* ---------------------------------------------------------------- decoded weights
 * P:36 / P:131: each element is the coefficient-weighted sum of its bits,
 * w[e] = sum_t c_t beta_t[e], c_t = s r^t + b from the stored fp16 s, b and R[r_idx]
 * (Eq. 4).  fp64, t in increasing order.  Used by the GEMV oracle (O-Y).               */
void oracle_decode_matrix(const uint32_t* planes, const uint16_t* s16, const uint16_t* b16, const uint8_t* r_idx,
                          int M, int N, int K, int G, int n_ratio, double* W_out) {
  const int NG = N / G, WPG = G / 32;
  double R[256];
  oracle_ratio_set(n_ratio, R);
  for (long q = 0; q < (long)M * NG; ++q) {
    long r = q / NG, g = q % NG;
    double c[OR_MAX_K];
    oracle_coefficients(R[r_idx[q]], oracle_fp16_to_double(s16[q]), oracle_fp16_to_double(b16[q]), K, c);
    const uint32_t* pl = planes + q * (long)K * WPG;
    for (int e = 0; e < G; ++e) {
      double w = 0.0;
      for (int t = 0; t < K; ++t)
        if ((pl[t * WPG + e / 32] >> (e % 32)) & 1u) w = w + c[t];
      W_out[r * (long)N + g * G + e] = w;
    }
  }
}

/* ---------------------------------------------------------------- O-Y GEMV (decode-then-dot)
 * The plain definition the SBVR kernel must reproduce:
 * y_r = sum_c w_dec[r,c] x_dec[c] in fp64, c in increasing order.  Rows may be a sample
 * (row_ids) so full-size layers can be checked one output at a time.                  */
void oracle_gemv_rows(const uint32_t* planes, const uint16_t* s16, const uint16_t* b16, const uint8_t* r_idx,
                      int M, int N, int K, int G, int n_ratio, const double* x_dec, const int32_t* row_ids,
                      int n_rows, double* y) {
  const int NG = N / G, WPG = G / 32;
  double R[256];
  oracle_ratio_set(n_ratio, R);
  (void)M;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int i = 0; i < n_rows; ++i) {
    long r = row_ids[i];
    double acc = 0.0;
    for (int g = 0; g < NG; ++g) {
      long q = r * NG + g;
      double c[OR_MAX_K];
      oracle_coefficients(R[r_idx[q]], oracle_fp16_to_double(s16[q]), oracle_fp16_to_double(b16[q]), K, c);
      const uint32_t* pl = planes + q * (long)K * WPG;
      for (int e = 0; e < G; ++e) {
        double w = 0.0;
        for (int t = 0; t < K; ++t)
          if ((pl[t * WPG + e / 32] >> (e % 32)) & 1u) w = w + c[t];
        acc = acc + w * x_dec[g * G + e];
      }
    }
    y[i] = acc;
  }
}

/* ---------------------------------------------------------------- O-P popcount partials
 * the AND/popcount inner product decomposes into the integers
 * P[t][j] = #{e : beta_t[e] = 1 and d_j[e] = 1} (here an element loop, NOT popcount)
 * and T[t] = sum_e beta_t[e] z[e].  Output P [n_rows][NG][K][l], T [n_rows][NG][K].   */
void oracle_partials_rows(const uint32_t* planes, const int32_t* z, const uint32_t* xplanes, int N, int K, int G,
                          int l, const int32_t* row_ids, int n_rows, int32_t* P, int32_t* T) {
  const int NG = N / G, WPG = G / 32;
  for (int i = 0; i < n_rows; ++i) {
    long r = row_ids[i];
    for (int g = 0; g < NG; ++g) {
      const uint32_t* pl = planes + (r * NG + g) * (long)K * WPG;
      const uint32_t* xp = xplanes + (long)g * l * WPG;
      for (int t = 0; t < K; ++t) {
        int32_t tt = 0;
        for (int e = 0; e < G; ++e)
          if ((pl[t * WPG + e / 32] >> (e % 32)) & 1u) tt += z[g * G + e];
        T[((long)i * NG + g) * K + t] = tt;
        for (int j = 0; j < l; ++j) {
          int32_t cnt = 0;
          for (int e = 0; e < G; ++e) {
            int bw = (pl[t * WPG + e / 32] >> (e % 32)) & 1u;
            int bx = (xp[j * WPG + e / 32] >> (e % 32)) & 1u;
            cnt += bw & bx;
          }
          P[(((long)i * NG + g) * K + t) * l + j] = cnt;
        }
      }
    }
  }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ randomized Hadamard rotation
 * PAPER.md P:255 (§4.5): weights are rotated by a randomized Hadamard transform before quantization
 * to Gaussianize them and suppress outliers.  Reading (A21): block-diagonal rotation along
 * the inner dimension N with blocks of b = 2^k columns, Q = H_b D / sqrt(b), D = diag(signs) (the
 * random +-1 draws are an input), H_b the Sylvester-Hadamard matrix, H_b[i][k] = (-1)^popcount(i & k).
 * Plain definition: y[i] = sum_k H_b[i][k] * signs[k] * x[k] / sqrt(b), an O(b^2) matrix-vector
 * product per block (no butterflies), fp64. */
void oracle_hadamard_rows(const double* X, double* Y, int rows, int N, int b, const int8_t* signs) {
  const double inv = 1.0 / sqrt((double)b);
#pragma omp parallel for schedule(static)
  for (long r = 0; r < rows; ++r) {
    for (int blk = 0; blk < N / b; ++blk) {
      const double* x = X + (size_t)r * N + (size_t)blk * b;
      const int8_t* sg = signs + (size_t)blk * b;
      double* y = Y + (size_t)r * N + (size_t)blk * b;
      for (int i = 0; i < b; ++i) {
        double acc = 0.0;
        for (int k = 0; k < b; ++k) {
          const double h = (__builtin_popcount((unsigned)(i & k)) & 1) ? -1.0 : 1.0;
          acc += h * (double)sg[k] * x[k];
        }
        y[i] = acc * inv;
      }
    }
  }
}

/* ------------------------------------------------------------------ O-PF prefill: FP16 decompression + GEMM
 * PAPER.md P:279 (§5.1): "we design a prefill kernel that decompresses SBVR weights into FP16 and transfers
 * the recovered weight segments to tensor cores for GEMM computation".  The paper does not say how the FP16
 * value is formed; reading A25: the coefficients of Eq. 4 are formed in fp32,
 *     c32_t = fmaf(s, (float) r^t, b)        (r^t by repeated fp64 multiplication, as oracle_coefficients)
 * rounded to fp16 (c16_t, round to nearest even), and the element is summed in fp16 arithmetic in plane order,
 *     w16 = fl16( ... fl16(fl16(0 + beta_0 c16_0) + beta_1 c16_1) ... + beta_{K-1} c16_{K-1})
 * (each partial sum of two fp16 values is exact in fp64 and rounded once).  The GEMM is the plain definition
 * y[tau][r] = sum_e fp64(w16[r][e]) * fp64(x16[tau][e]), e increasing, fp64.                                */
static void prefill_coefs16(double r, uint16_t s16, uint16_t b16, int K, double* c16) {
  const float s = (float)oracle_fp16_to_double(s16), b = (float)oracle_fp16_to_double(b16);
  double p = 1.0;
  for (int t = 0; t < K; ++t) {
    const float c32 = fmaf(s, (float)p, b);
    c16[t] = oracle_fp16_to_double(oracle_fp16_bits((double)c32));
    p = p * r;
  }
}

static uint16_t prefill_element16(const uint32_t* pl, int WPG, int e, const double* c16, int K) {
  double acc = 0.0;
  for (int t = 0; t < K; ++t)
    if ((pl[t * WPG + e / 32] >> (e % 32)) & 1u) acc = oracle_fp16_to_double(oracle_fp16_bits(acc + c16[t]));
  return oracle_fp16_bits(acc);
}

void oracle_prefill_decode_fp16(const uint32_t* planes, const uint16_t* s16, const uint16_t* b16,
                                const uint8_t* r_idx, int M, int N, int K, int G, int n_ratio, uint16_t* W16) {
  const int NG = N / G, WPG = G / 32;
  double R[256];
  oracle_ratio_set(n_ratio, R);
  for (long q = 0; q < (long)M * NG; ++q) {
    const long r = q / NG, g = q % NG;
    double c16[OR_MAX_K];
    prefill_coefs16(R[r_idx[q]], s16[q], b16[q], K, c16);
    const uint32_t* pl = planes + q * (long)K * WPG;
    for (int e = 0; e < G; ++e) W16[r * (long)N + g * G + e] = prefill_element16(pl, WPG, e, c16, K);
  }
}

void oracle_prefill_rows(const uint32_t* planes, const uint16_t* s16, const uint16_t* b16, const uint8_t* r_idx,
                         int M, int N, int K, int G, int n_ratio, const uint16_t* X16, int T, const int32_t* row_ids,
                         int n_rows, double* Y) {
  const int NG = N / G, WPG = G / 32;
  double R[256];
  oracle_ratio_set(n_ratio, R);
  (void)M;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int i = 0; i < n_rows; ++i) {
    const long r = row_ids[i];
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    for (int g = 0; g < NG; ++g) {
      const long q = r * NG + g;
      double c16[OR_MAX_K];
      prefill_coefs16(R[r_idx[q]], s16[q], b16[q], K, c16);
      const uint32_t* pl = planes + q * (long)K * WPG;
      for (int e = 0; e < G; ++e) w[g * G + e] = oracle_fp16_to_double(prefill_element16(pl, WPG, e, c16, K));
    }
    for (int tau = 0; tau < T; ++tau) {
      const uint16_t* x = X16 + (size_t)tau * N;
      double acc = 0.0;
      for (int e = 0; e < N; ++e) acc = acc + w[e] * oracle_fp16_to_double(x[e]);
      Y[(size_t)tau * n_rows + i] = acc;
    }
    free(w);
  }
}
