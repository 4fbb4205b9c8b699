/*
 * sbvr.h -- C-ABI of libsbvr: the SBVR (arXiv 2509.18172) hot path on NVIDIA B200 (sm_100a).
 *
 * The core calls follow the paper's problem statement: encode
 * weights offline, convert activations online, and run the GEMV directly on the SBVR
 * format without decompressing it.
 *
 *   sbvr_encode_weights   Section 4.2, Eq. 4-11, Algorithm 1, bit assignment
 *   sbvr_encode_vector    Section 4.3, Eq. 12
 *   sbvr_gemv             Section 4.4: y = W x on SBVR weights, x either fp16 or SBVR
 *   sbvr_gemv_batched     the same for T <= 256 activation vectors sharing weight fetches
 *   sbvr_gemv_group       several independent batch-1 GEMVs (a decoder layer's projections) in one launch
 *   sbvr_prefill          Section 5.1: the prefill GEMM on FP16-decompressed weights (tensor cores)
 *
 * Conventions (all calls):
 *  - Plain C types only.  "Device" pointers are CUDA global-memory pointers on the current
 *    device; "host" pointers are CPU memory.  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - Ownership: the library never allocates, frees or retains memory.  Callers query sizes
 *    (sbvr_weights_bytes, sbvr_gemv_workspace_bytes), allocate, and pass raw pointers.
 *  - Execution: every device call only enqueues work on `stream`; it never synchronizes the
 *    device, and it is CUDA-graph capturable.  Arguments are validated before any launch.
 *  - Errors: every call returns an sbvr_status.  SBVR_OK = success.  Validation failures
 *    return SBVR_ERR_INVALID_ARG / _SHAPE / _UNSUPPORTED / _ALIGNMENT / _WORKSPACE without
 *    enqueuing anything; a failed launch returns SBVR_ERR_CUDA.  sbvr_last_error() gives a
 *    thread-local human-readable detail.  No C++ exception crosses this ABI.
 *  - Determinism: no floating-point atomics; reduction orders are fixed for a given device
 *    (SM count).  Integer outputs (planes, partials) are bit-exact.
 *
 * ---------------------------------------------------------------------------------------
 * Canonical (interchange) layouts -- what tests compare against the oracle:
 *   planes  [M][N/G][K][G/32] uint32, bit i of word w = element 32w+i of the group, LSB first
 *   meta    s16, b16 [M][N/G] IEEE fp16 bit patterns; r_idx [M][N/G] uint8 (index into R)
 *
 * Device weight layout (written by sbvr_encode_weights, read by the GEMV kernels; G = 128):
 *   Rows are cut into row blocks of 128 rows (M % 16 == 0; the last block holds M % 128 rows
 *   when M is not a multiple of 128).  A *unit* is (row block rb, group g), stored as ONE
 *   contiguous record of R = rows-in-block rows:
 *       [R x 16K bytes: bit-planes][R x 4 B: scale/bias][R x 1 B: ratio index]
 *   Units are ordered rb-major (unit index rb*NG + g, NG = N/128); full blocks are 128*(16K+5)
 *   bytes each, the tail block's NG units follow.  Total = M*N*K/8 + 5*M*N/128 bytes.
 *   Row r of a unit holds K 16-byte chunks; chunk t = words c = 0..3 of plane t (elements
 *   32c..32c+31 of the group) and is stored at chunk position t ^ swz(r), swz(r) = (r>>2)&1 for
 *   K = 2 or 6, (r>>1)&3 for K = 4, r&7 for K = 8, 0 otherwise (so eight consecutive rows'
 *   16-byte loads of one plane hit eight distinct shared-memory bank groups).  One GEMV thread
 *   owns one row = one tensor-memory lane.
 *   scale/bias word r = fp16 s (bits 0-15) | fp16 b (bits 16-31); ratio-index byte r = uint8
 *   index into R.
 *   ratio_pow [n_ratio][K] fp32 = r_i^t (repeated multiplication in fp64, rounded to fp32).
 *   SBVR_META_INDEXED: the same records with the 5-byte meta replaced by one byte per row:
 *       [R x 16K bytes: bit-planes][R x 1 B: coefficient-table index]   (total M*N*K/8 + M*N/128 bytes)
 *   and the coefficient table in coef_table (2 KB).
 *
 * Device activation layout (SBVR-x, written by sbvr_encode_vector):
 *   planes [T][N/G][l][G/32] uint32 (same bit order as the weights), scales [T][N/G] fp32.
 *   fp16-x: x is uint16_t (IEEE fp16 bits) [T][N].
 */
#ifndef SBVR_H_
#define SBVR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBVR_ABI_VERSION 2

typedef enum {
  SBVR_OK = 0,
  SBVR_ERR_INVALID_ARG = 1,  /* null pointer, out-of-range scalar */
  SBVR_ERR_SHAPE = 2,        /* M % 16, N % G, x.N != W.N, group sizes differ, T out of range */
  SBVR_ERR_UNSUPPORTED = 3,  /* K, l, G or config outside what this build implements */
  SBVR_ERR_ALIGNMENT = 4,    /* device pointer not 16-byte aligned */
  SBVR_ERR_CUDA = 5,         /* a CUDA launch or attribute query failed */
  SBVR_ERR_WORKSPACE = 6     /* workspace missing or too small */
} sbvr_status;

typedef enum { SBVR_F32 = 0, SBVR_F16 = 1, SBVR_BF16 = 2 } sbvr_dtype;
/* Activation kinds.  SBVR_ACT_FP16_Q: fp16 x (data = uint16_t[N]) that the GEMV converts to SBVR-x itself, in its
 * prologue, with exactly the arithmetic of sbvr_encode_vector (Eq. 12, l bits) -- the result is bit-identical to
 * sbvr_encode_vector + sbvr_gemv on SBVR-x, without the separate conversion launch.  T = 1, MMA kernel, K 2..4. */
typedef enum { SBVR_ACT_FP16 = 0, SBVR_ACT_SBVR = 1, SBVR_ACT_FP16_Q = 2 } sbvr_act_kind;

/* GEMV algorithm selector for sbvr_gemv_ex / sbvr_debug_partials.
 *  AUTO  : the fastest implemented kernel for the activation kind and batch (measured; SBVR-x: MMA,
 *          which switches to its z-column form for T >= 3).
 *  POPC  : the paper's formulation, CUDA-core AND + __popc + coefficient FMAs.
 *  TC    : bit-sliced popcount on the 5th-generation tensor cores: A = plane & 0x01010101<<s in
 *          tensor memory, B = d_j bit-sliced x 2^(7-s) in shared memory, tcgen05.mma kind::i8
 *          M=128 N=8T K=32, which counts popc(beta_t & d_j) for 128 rows x 8 planes x T tokens.
 *  MMA   : the same bit-sliced popcount with warp-level mma.sync.m16n8k32.u8 (16 rows x 8 planes
 *          per instruction), the faster issue rate at batch 1.  For T >= 3 SBVR-x tokens it uses the
 *          z-column form: A = the plane bits themselves (u8 0/1), B = the tokens' int8 z = sum_j
 *          alpha_j d_j (s8, 8 tokens as the 8 MMA columns), so the accumulator holds
 *          T_t = sum_j alpha_j popc(beta_t & d_j) per token directly (same integers).
 *  ZT    : batches on tcgen05 in the z-column form: A = the weight-plane bits as bytes 0/1 in tensor
 *          memory (M = 128 rows, K = 32 elements), B = the tokens' int8 z = sum_j alpha_j d_j (s8, N = up to 32
 *          tokens), kind::i8, so T_t = sum_e beta_t[e] z_e = sum_j alpha_j popc(beta_t & d_j) lands in tensor
 *          memory for 128 rows x N tokens per instruction; one weight pass per 32 tokens (tensor cores
 *          amortise the weight decoding over the tokens).  SBVR-x, K <= 4.  AUTO picks it for T >= 12 (measured crossover vs MMA).
 *  PIPE  : the MMA formulation in a persistent warp-specialised kernel (producer warp + CTA-wide TMA
 *          ring, dynamically ticketed work items, deterministic split-K combine); batch 1, SBVR-x.
 *          Explicit only: measured slower than MMA on the Llama-3-8B step.          */
typedef enum { SBVR_ALGO_AUTO = 0, SBVR_ALGO_POPC = 1, SBVR_ALGO_TC = 2, SBVR_ALGO_MMA = 3, SBVR_ALGO_PIPE = 4,
               SBVR_ALGO_ZT = 5 } sbvr_algo;

/* Offline encoder knobs (SURVEY §8c.3 readings A1, A4). */
typedef struct {
  int32_t K;             /* weight bit-planes; 1..6 supported by the encoder, 2..4 targeted */
  int32_t group_size;    /* elements per group along N; 128 only in this build */
  int32_t n_ratio;       /* |R|, even, 2..64 (R = two linspaces over [-1,-0.5] and [0.5,1]) */
  int32_t n_scale;       /* |S|, 1..4096 */
  int32_t n_bias;        /* |B|, 1..4096 */
  double s_min_factor;   /* s_min = s_min_factor * q95(D); 2.0 = paper Eq. 10 */
  int32_t strict;        /* 1 = fp64 search bit-identical to the oracle; 0 = fast (sbvr_encode_weights only): every
                            entry's MSE in fp32, then the strict fp64 MSE of the entries within a margin of the fp32
                            best and their strict arg-min in entry order (SURVEY §8c.5 contract: the choice's fp64
                            MSE <= (1 + 1e-6) x the strict best; planes = the nearest assignment for the chosen
                            coefficients, computed in fp64 as in strict mode) */
} sbvr_encode_config;

/* Per-group coefficient metadata of a weight buffer. */
typedef enum {
  SBVR_META_GROUP = 0,   /* every group stores fp16 s, fp16 b and a u8 ratio index (5 B per group) */
  SBVR_META_INDEXED = 1  /* every group stores a u8 index into a per-matrix coefficient table (1 B per group):
                            "a coefficient cache containing all coefficient sets required for decoding, as well
                            as a coefficient index" */
} sbvr_meta_kind;

/* Encoded weights (device pointers, caller-owned; sizes from sbvr_weights_bytes / sbvr_weights_bytes_ex). */
typedef struct {
  int32_t M, N, K, group_size, n_ratio;
  uint8_t* data;         /* packed units (layout above), 16-byte aligned */
  float* ratio_pow;      /* [n_ratio][K], 16-byte aligned */
  int32_t meta_kind;     /* sbvr_meta_kind; SBVR_META_GROUP unless the weights come from the indexed encoder */
  uint32_t* coef_table;  /* SBVR_META_INDEXED: [1 + 2 * 256] u32 -- word 0 = number of entries n (1..256), then
                            per entry (fp16 s | fp16 b << 16, ratio index); NULL for SBVR_META_GROUP */
} sbvr_weights;

/* One activation descriptor; for T vectors the buffers hold T contiguous vectors. */
typedef struct {
  int32_t kind;          /* sbvr_act_kind */
  int32_t N, group_size; /* must equal the weights' N and group_size */
  int32_t l;             /* SBVR-x activation bit-width, 2..8 (l = 8) */
  const void* data;      /* FP16: uint16_t[T][N];  SBVR: uint32_t[T][N/G][l][G/32] */
  const float* scales;   /* SBVR: [T][N/G]; ignored for FP16 */
} sbvr_act;

int32_t sbvr_abi_version(void);
const char* sbvr_status_string(sbvr_status s);
const char* sbvr_last_error(void);

/* Byte sizes of the two weight buffers for an M x N matrix with K planes. */
sbvr_status sbvr_weights_bytes(int32_t M, int32_t N, int32_t K, int32_t group_size, int32_t n_ratio,
                               size_t* data_bytes, size_t* ratio_pow_bytes);

/* sbvr_encode_weights -- P:150-233.  For every group of G consecutive elements of every row
 * of W (device, row-major [M][N], dtype F32/F16/BF16), build the candidate sets of Eq. 5-11,
 * run Algorithm 1's exhaustive MSE search over R x S x B (R outer, S middle, B inner, strict
 * '<'), assign each element the mask of its nearest subset sum, and write data and
 * ratio_pow of `out` (whose M, N, K, group_size, n_ratio must match
 * cfg / the arguments).  group_mse (nullable, device, [M][N/G] fp64, row-major) receives each
 * group's winning MSE.  Groups run in parallel on the GPU. */
sbvr_status sbvr_encode_weights(const sbvr_encode_config* cfg, const void* W, int32_t dtype, int32_t M,
                                int32_t N, const sbvr_weights* out, double* group_mse, void* stream);

/* Byte sizes for either meta kind (sbvr_weights_bytes = SBVR_META_GROUP); table = bytes of coef_table. */
sbvr_status sbvr_weights_bytes_ex(int32_t M, int32_t N, int32_t K, int32_t group_size, int32_t n_ratio,
                                  int32_t meta_kind, size_t* data_bytes, size_t* ratio_pow_bytes, size_t* table_bytes);

/* sbvr_encode_weights_indexed -- SBVR weights in the table + index format (P:233's cache of previously
 * selected r, s, b; reading A23): (1) Algorithm 1, exactly as sbvr_encode_weights, on min(n_table, groups) evenly
 * spaced sample groups (row-major group q_i = floor(i * groups / n_sample)); (2) the coefficient table = their
 * winning (r, s, b), duplicates dropped, in sample order; (3) every group takes the table entry of least MSE
 * (strict '<' in table order) and its bits are assigned for that entry.  n_table: 1..256.  out must have
 * meta_kind = SBVR_META_INDEXED, data sized by sbvr_weights_bytes_ex and coef_table set.  group_mse as in
 * sbvr_encode_weights.  workspace: device scratch of >= 8 * n_table bytes.  Strict fp64, bit-identical with the
 * oracle; all work on `stream`. */
sbvr_status sbvr_encode_weights_indexed(const sbvr_encode_config* cfg, int32_t n_table, const void* W, int32_t dtype,
                                        int32_t M, int32_t N, const sbvr_weights* out, double* group_mse,
                                        void* workspace, size_t ws_bytes, void* stream);

/* sbvr_encode_weights_cached -- the encode-time coefficient cache of P:233 (§4.2 and its footnote):
 * "we maintain a cache of previously selected variables r, s, and b ... check the cache ... before
 * exploring the entire search space"; "if the error from the cached values is below this moving average
 * [of the quantization error], the cached values are used".  Reading A22: per row, groups left to right
 * (deterministic; rows run in parallel on the GPU), an MRU cache of up to cache_size (0..64) (r, s, b)
 * triples, hit when the best cached MSE (strict '<', MRU order) < the moving average
 * ema = (1-ema_alpha) ema + ema_alpha mse (initialised to the row's first full-search MSE); a miss runs
 * Algorithm 1 exactly as sbvr_encode_weights and puts its winner in front.  Outputs as
 * sbvr_encode_weights; group_hit (nullable, device, [M][N/G] uint8) = 1 for groups that took a cached set.
 * cache_size = 0 gives exactly sbvr_encode_weights' result. */
sbvr_status sbvr_encode_weights_cached(const sbvr_encode_config* cfg, int32_t cache_size, double ema_alpha,
                                       const void* W, int32_t dtype, int32_t M, int32_t N, const sbvr_weights* out,
                                       double* group_mse, uint8_t* group_hit, void* stream);
/* sbvr_encode_vector -- P:235-243, Eq. 12.  x: device fp16 bits [T][N].  Per group of G:
 * s_x = absmax/(2^(l-1)-1) (fp32 IEEE), z = clamp(rne(x/s_x)), planes = l-bit two's
 * complement of z (plane l-1 = sign, weight -2^(l-1) s_x).  Outputs (device):
 * planes_out [T][N/G][l][G/32] uint32, scales_out [T][N/G] fp32.  All-zero group -> s_x = 0. */
sbvr_status sbvr_encode_vector(const uint16_t* x, int32_t T, int32_t N, int32_t group_size, int32_t l,
                               uint32_t* planes_out, float* scales_out, void* stream);

/* Workspace for the GEMV kernels (cross-CTA partial-sum slots and flags for row blocks split
 * over several CTAs).  Before its first use a workspace must be initialised with
 * sbvr_workspace_init (fills it with 0xFF bytes: "slot empty / flag clear"); every GEMV leaves
 * it in that state again.  One workspace must not be used by two GEMVs running concurrently on
 * different streams. */
sbvr_status sbvr_gemv_workspace_bytes(const sbvr_weights* w, int32_t T, size_t* bytes);
sbvr_status sbvr_workspace_init(void* workspace, size_t bytes, void* stream);

/* sbvr_gemv -- P:245-251.  y[M] (device fp32) = W x with W in SBVR form, never decompressed.
 * SBVR-x: y_r = sum_g s_x,g sum_t c_t sum_j alpha_j popc(beta_t & d_j), c_t = s r^t + b
 * (alpha_j = 2^j, alpha_{l-1} = -2^(l-1)); fp16-x: y_r = sum_g sum_t c_t sum_e beta_t[e] x_e.
 * Popcount partials are exact integers; the float part accumulates in fp32. */
sbvr_status sbvr_gemv(const sbvr_weights* w, const sbvr_act* x, float* y, void* workspace, size_t ws_bytes,
                      void* stream);

/* sbvr_gemv_batched -- T (1..256) activation vectors in one descriptor (T decode streams, or a prefill chunk);
 * Y [T][M] fp32.  The kernels loop over token passes (ZT: 32 tokens per weight pass; MMA: 8). */
sbvr_status sbvr_gemv_batched(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* Y, void* workspace,
                              size_t ws_bytes, void* stream);

/* sbvr_gemv_chain -- sbvr_gemv_batched plus a hint naming the weights of the GEMV that the caller launches next on
 * the same stream (e.g. the next projection of a decoder layer, or the next layer's first).  Results are identical
 * to sbvr_gemv_batched; the hint only moves data: once a CTA has issued its last weight copy, it prefetches into
 * L2 the first unit records that CTA index will copy first in a GEMV over next_w, so the next launch's pipeline
 * fill hits L2 instead of waiting on HBM (B200 126 MB L2).  next_w may be NULL (= sbvr_gemv_batched); it is only
 * read as addresses and shape (SBVR_META_GROUP weights; ignored for other kinds). */
sbvr_status sbvr_gemv_chain(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* Y, void* workspace,
                            size_t ws_bytes, const sbvr_weights* next_w, void* stream);

/* sbvr_gemv_to_peers -- the row-sharded multi-GPU GEMV with the all-gather fused into its epilogue (north star
 * "row-sharded multi-GPU path ... joins y").  W is this rank's row shard (rows
 * [y_row_offset, y_row_offset + W.M) of an M_full-row matrix); every y value the kernel produces is stored, over
 * NVLink, into each of the n_peers (1..8) buffers peer_y[j] -- device pointers, typically the ranks' symmetric-
 * memory full-y buffers (own rank included), each [T][M_full] fp32 -- at [tau][y_row_offset + row], so no
 * separate all-gather runs.  peer_y is a HOST array of device pointers.  The caller orders the stores before any
 * read of the full y on another rank with a signal-pad barrier (dist.py).  Same arithmetic, partition and
 * determinism as sbvr_gemv_batched on the MMA kernel.  Errors: as sbvr_gemv; SBVR_ERR_SHAPE when the shard does
 * not fit M_full. */
sbvr_status sbvr_gemv_to_peers(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* const* peer_y,
                               int32_t n_peers, int32_t y_row_offset, int32_t M_full, void* workspace, size_t ws_bytes,
                               void* stream);

/* sbvr_gemv_group -- several INDEPENDENT batch-1 GEMVs y_p = W_p x_p (the SBVR-x AND+popcount form of
 * sbvr_gemv) in one persistent launch, e.g. the projections of a decoder layer whose inputs are all available
 * (grouped GEMV).  The problems' unit records form one work sequence that is split evenly over the CTAs, so the
 * fixed costs of a launch (pipeline fill, split-K combine, tail, launch boundary) are paid once per group instead
 * of once per matrix, and the next matrix's weights stream in while the current one finishes.
 *   probs: HOST array of n (1..SBVR_GROUP_MAX) problems; each holds a weights and an activation descriptor (by
 *          value) and y (device fp32 [M]).  No problem may write a buffer another problem reads (y's must not
 *          overlap x, scales or weights); y's must not overlap each other.
 *   Supported: SBVR_ACT_SBVR activations (T = 1, the same l for all), SBVR_META_GROUP weights, K in 2..4 and equal
 *   for all problems, M % 128 == 0 (SBVR_ERR_UNSUPPORTED / SBVR_ERR_SHAPE otherwise).  SBVR_ACT_FP16_Q activations
 *   (all problems): the kernel converts every x itself (Eq. 12, bit-identical to sbvr_encode_vector) with a
 *   grid-wide arrival count between conversion and use -- the grid is sized to the co-resident CTA count the
 *   driver reports, so it must not share the GPU with another kernel that waits on this one.
 *   workspace: >= sbvr_gemv_group_workspace_bytes bytes, initialised once with sbvr_workspace_init and left at
 *   rest by every call; not shared with a concurrently running GEMV.
 * Arithmetic and per-band reduction order are those of sbvr_gemv's MMA kernel; y is deterministic. */
#define SBVR_GROUP_MAX 8
typedef struct {
  sbvr_weights w;
  sbvr_act x;
  float* y;
} sbvr_gemv_problem;
sbvr_status sbvr_gemv_group_workspace_bytes(const sbvr_gemv_problem* probs, int32_t n, size_t* bytes);
sbvr_status sbvr_gemv_group(const sbvr_gemv_problem* probs, int32_t n, void* workspace, size_t ws_bytes, void* stream);

/* sbvr_gemv_group_to_peers -- sbvr_gemv_group over this rank's row shards with the all-gather fused into the
 * epilogue (north star "row-sharded multi-GPU path ... joins y"): every y value of problem i is stored
 * into each of the n_peers (1..8) buffers peer_y[i * n_peers + j] -- device pointers, typically every rank's
 * symmetric-memory full y of problem i, [M_full[i]] fp32 each -- at row y_row_offset[i] + row; probs[i].y is ignored.
 * peer_y, y_row_offset and M_full are HOST arrays.  The caller orders the stores before any read of a full y on
 * another rank (signal-pad barrier, dist.py).  Same arithmetic, partition and determinism as sbvr_gemv_group; the
 * same restrictions.  Errors: as sbvr_gemv_group; SBVR_ERR_SHAPE when a shard does not fit its M_full. */
sbvr_status sbvr_gemv_group_to_peers(const sbvr_gemv_problem* probs, int32_t n, float* const* peer_y, int32_t n_peers,
                                     const int32_t* y_row_offset, const int32_t* M_full, void* workspace,
                                     size_t ws_bytes, void* stream);

/* sbvr_gemv_ex -- as sbvr_gemv_batched with an explicit algorithm (sbvr_algo). */
sbvr_status sbvr_gemv_ex(const sbvr_weights* w, const sbvr_act* X, int32_t T, float* Y, void* workspace,
                         size_t ws_bytes, int32_t algo, void* stream);

/* sbvr_hadamard_rows -- randomized Hadamard rotation, P:255 (Section 4.5): "rotate the weights with a
 * randomized Hadamard transform to Gaussianize them and suppress outliers" before encoding (and the
 * activations with the same orthogonal Q, since W x = (W Q^T)(Q x)).  Reading A21: block-diagonal along
 * N; every block of `block` consecutive columns of every row becomes
 *     Y[r, blk*b + i] = sum_k (-1)^popcount(i & k) * signs[blk*b + k] * X[r, blk*b + k] / sqrt(b).
 * X, Y: device, row-major [rows][N], dtype SBVR_F32 or SBVR_F16 (fp32 arithmetic); Y == X allowed
 * (in place).  signs: device int8 [N], each +1 or -1 (the random diagonal D, caller-drawn).  block: a
 * power of two in 32..1024 with N % block == 0 (SBVR_ERR_UNSUPPORTED / SBVR_ERR_SHAPE otherwise).
 * Buffers 16-byte aligned. */
sbvr_status sbvr_hadamard_rows(const void* X, void* Y, int32_t dtype, int32_t rows, int32_t N, int32_t block,
                               const int8_t* signs, void* stream);
/* sbvr_prefill -- the prefill GEMM of PAPER.md P:279 (§5.1): "a prefill kernel that decompresses SBVR
 * weights into FP16 and transfers the recovered weight segments to tensor cores for GEMM computation".
 *   Y[tau][r] = sum_e w16[r][e] * X[tau][e]      (fp32 accumulation on tcgen05.mma kind::f16)
 * with w16 the FP16 decompression of reading A25: c16_t = fp16(fmaf(s, r^t, b)) and
 * w16 = fl16(... fl16(beta_0 c16_0) + ... + beta_{K-1} c16_{K-1}) in plane order -- bit-identical to the
 * oracle's O-PF decode.  One pass over the weights per 256 tokens.
 *   w          SBVR_META_GROUP weights, K = 1..4, any M (multiple of 16), N multiple of 128 (device)
 *   X          device, fp16 bit patterns [T][N] row-major (8-byte aligned); read-only
 *   T          tokens, >= 0 (0: nothing enqueued); any size (passes of 256)
 *   Y          device, fp32 [T][M] row-major (4-byte aligned); every element written
 *   workspace  device, 256-byte aligned, >= sbvr_prefill_workspace_bytes(w, T); initialised once with
 *              sbvr_workspace_init and left at rest by every call (the token relayout scratch inside it is
 *              overwritten); one call at a time per workspace.
 * Errors: SBVR_ERR_UNSUPPORTED (indexed meta, K > 4), _SHAPE (T < 0), _ALIGNMENT, _WORKSPACE, _CUDA. */
sbvr_status sbvr_prefill_workspace_bytes(const sbvr_weights* w, int32_t T, size_t* bytes);
sbvr_status sbvr_prefill(const sbvr_weights* w, const uint16_t* X, int32_t T, float* Y, void* workspace,
                         size_t ws_bytes, void* stream);

/* Test-only: the integer popcount partials P[m][g][t][j] = popc(beta_t & d_j) over the group,
 * int32 [M][N/G][K][l] row-major (device), computed by the kernel `algo` (POPC, TC or MMA) from an
 * SBVR-x activation (T = 1). */
sbvr_status sbvr_debug_partials(const sbvr_weights* w, const sbvr_act* x, int32_t algo, int32_t* P, void* stream);

/* Test-only: the exact integers T_t = sum_e beta_t[e] z_e of the ZT kernel (before any float arithmetic),
 * int32 [M][N/G][K][T] row-major (device), SBVR-x activation with T (1..32) tokens. */
sbvr_status sbvr_debug_zt_sums(const sbvr_weights* w, const sbvr_act* x, int32_t T, int32_t* Tsum, void* stream);

/* Host-side layout transforms (host memory on both sides, no device work).  canonical planes
 * [M][N/G][K][G/32], s16/b16/r_idx [M][N/G]  <->  the packed device-layout image `data`
 * (size as sbvr_weights_bytes).  Bit-exact inverses of each other. */
sbvr_status sbvr_pack_canonical(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint32_t* planes_canon,
                                const uint16_t* s16, const uint16_t* b16, const uint8_t* r_idx, uint8_t* data);
sbvr_status sbvr_unpack_canonical(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint8_t* data,
                                  uint32_t* planes_canon, uint16_t* s16, uint16_t* b16, uint8_t* r_idx);

/* Indexed-format host transforms: canonical planes [M][N/G][K][G/32] + table index [M][N/G] u8 <-> the packed
 * SBVR_META_INDEXED image `data` (size from sbvr_weights_bytes_ex).  Bit-exact inverses. */
sbvr_status sbvr_pack_indexed(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint32_t* planes_canon,
                              const uint8_t* idx, uint8_t* data);
sbvr_status sbvr_unpack_indexed(int32_t M, int32_t N, int32_t K, int32_t group_size, const uint8_t* data,
                                uint32_t* planes_canon, uint8_t* idx);

/* Write w->ratio_pow (device) for w->n_ratio, w->K (used when weights arrive via pack). */
sbvr_status sbvr_fill_ratio_table(const sbvr_weights* w, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SBVR_H_ */
