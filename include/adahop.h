/*
 * adahop.h — C ABI of the B200-native AdaHOP MXFP4 linear (arXiv 2604.02525).
 *
 * Citations: P:<n> = line n of the paper's LaTeX source; the section,
 * equation or table is named beside each one.
 *
 * The library computes, for one matmul C = A·B of a linear layer (P:72-79,
 * eq:forward / eq:backward_gw / eq:backward_gx):
 *   IHT:        C = Q(A H) · Q(H^T B)                        (eq:inner_hadamard)
 *   OE-Left:    C = Q(A_res H) · Q(H^T B) + A_out · B        (eq:oe_left)
 *   OE-Right:   C = Q(A H) · Q(H^T B_res) + A · B_out        (eq:oe_right)
 *   BF16:       C = A · B in BF16                            (AdaHOP-Lv2 CC)
 * H = blockwise normalised Walsh–Hadamard (block 32 along K); Q = MXFP4 (E2M1
 * elements, one E8M0 scale per 32 elements along K); A_out / B_out = the top-k rows of
 * A / columns of B chosen by FOID (variance of the first 64 elements).
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless a parameter says "host". Matrices are
 *    row-major with an explicit leading dimension (elements).
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default).
 *    The library never allocates, frees, or synchronises on the hot path; it is
 *    stateless apart from a per-device property cache, thread-safe, and every hot-path
 *    call is CUDA-graph capturable (k and shapes are host values; indices stay on device).
 *  - Ownership: the caller owns every buffer. Scratch comes from the caller's
 *    workspace `ws` of `ws_bytes` bytes (query with adahop_workspace_bytes); it must be
 *    256-byte aligned and must not be used by other work concurrently.
 *  - Errors: all argument/shape checks run on the host before any launch, so an error
 *    never leaves partial writes. A failed launch returns ADAHOP_E_CUDA. No exceptions
 *    cross the ABI, nothing is printed, nothing aborts.
 *  - Inputs must be finite (non-finite input is undefined behaviour).
 *  - Shape rules: K % 32 == 0 (else ADAHOP_E_SHAPE; no padding);
 *    had_block must be 32 (else ADAHOP_E_UNSUPPORTED); oe_k > rows/cols of the
 *    extracted operand clamps; oe_k == 0 means "no OE"; oe_k <= 256; the OE operand has at
 *    most 65536 stored rows (ADAHOP_E_UNSUPPORTED beyond: the FOID select merges the
 *    k-best of 16 blocks of 4096 rows) — e.g. up to 65536 tokens per GPU for an OE on the
 *    token dimension (dgrad OE-Left on G_Y, fwd OE-Left on X).
 *    Leading dimensions must keep every row 16-byte aligned.
 */
#ifndef ADAHOP_H_
#define ADAHOP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADAHOP_ABI_VERSION 2

typedef struct CUstream_st* adahop_stream_t; /* == cudaStream_t */

typedef enum {
  ADAHOP_OK = 0,
  ADAHOP_E_INVALID_ARG = 1,  /* null pointer, bad enum, bad leading dimension        */
  ADAHOP_E_SHAPE = 2,        /* K % 32 != 0, non-positive sizes, T % 32 in wgrad     */
  ADAHOP_E_UNSUPPORTED = 3,  /* had_block != 32, oe_k > 256, unsupported dtype       */
  ADAHOP_E_WORKSPACE = 4,    /* ws too small or misaligned                           */
  ADAHOP_E_CUDA = 5,         /* a CUDA launch / driver call failed                   */
  ADAHOP_E_NO_DEVICE = 6     /* no sm_100 device (the library has no CPU fallback)   */
} adahop_status_t;

/* Outlier pattern of a tensor as fed to the matmul. */
typedef enum {
  ADAHOP_PAT_INVALID = -1,   /* returned by adahop_majority_vote for an empty / invalid record */
  ADAHOP_PAT_NONE = 0,
  ADAHOP_PAT_ROW = 1,
  ADAHOP_PAT_COL = 2
} adahop_pattern_t;

/* Strategy (tab:strategy_summary). */
typedef enum {
  ADAHOP_IHT = 0,
  ADAHOP_OE_LEFT_IHT = 1,
  ADAHOP_OE_RIGHT_IHT = 2,
  ADAHOP_BF16 = 3
} adahop_strategy_t;

typedef enum { ADAHOP_DT_BF16 = 0, ADAHOP_DT_F32 = 1 } adahop_dtype_t;

/* The three matmuls of a linear layer. */
typedef enum { ADAHOP_PATH_FWD = 0, ADAHOP_PATH_DGRAD = 1, ADAHOP_PATH_WGRAD = 2 } adahop_path_t;

typedef struct {
  int32_t had_block;  /* Hadamard block along K; 32                         */
  int32_t oe_k;       /* extracted rows/cols; 64; 0 = no OE          */
  int32_t foid_probe; /* FOID probe length; 64                              */
  int32_t level;      /* 1 = AdaHOP-Lv1, 2 = AdaHOP-Lv2                 */
  float tau;          /* CV threshold; 2.0                                  */
  float eps;          /* CV stabiliser; 1e-8 ("small constant")               */
} adahop_params_t;

/* ---------------------------------------------------------------- host utilities */

/* Fill `p` (host) with the paper's defaults: 32, 64, 64, 1, 2.0, 1e-8. */
void adahop_default_params(adahop_params_t* p);
int32_t adahop_abi_version(void);
const char* adahop_status_string(adahop_status_t s);

/* tab:strategy_summary: CN,NN,CR,NR -> IHT; RN,RR -> OE-Left; RC,NC -> OE-Right;
 * CC -> OE-Right (level 1) or BF16 (level 2). Pure host function. */
adahop_strategy_t adahop_strategy_for_pair(adahop_pattern_t left, adahop_pattern_t right,
                                           int32_t level);

/* Strategies of the three matmuls of one linear from its tensors' calibrated patterns (host, pure;
 * §5.1 step 3). Patterns are detected on the tensors as stored — X [T x d_in],
 * W [d_out x d_in], G_Y [T x d_out] — and the fed operand pairs are
 *   fwd (X, W^T), dgrad (G_Y, W), wgrad (G_Y^T, X), with pattern(T^T) = swap(R <-> C)
 * (R8, pinned by Table 1's cross-path identities). Writes out[0..2] = the strategies of
 * {fwd, dgrad, wgrad} and, when fed_pairs is not NULL, fed_pairs[2 p], fed_pairs[2 p + 1] = the
 * fed (left, right) patterns of path p. Returns 0, or -1 for an invalid pattern / level. */
int32_t adahop_layer_strategies(adahop_pattern_t pat_x, adahop_pattern_t pat_w, adahop_pattern_t pat_gy,
                                int32_t level, adahop_strategy_t* out, adahop_pattern_t* fed_pairs);

/* Majority vote over per-step patterns; ties resolve R > C > N (R9).
 * `per_step` is a host array of n >= 1 pattern codes (0, 1, 2). Returns ADAHOP_PAT_INVALID for
 * a NULL array, n <= 0, or any code outside {0, 1, 2} (an input error, like the oracle's). */
adahop_pattern_t adahop_majority_vote(const int32_t* per_step, int32_t n);

/* Classification rule of App. A on already-reduced CVs (host, pure):
 * ROW if cv_col > tau, COL if cv_row > tau, larger wins when both, tie -> ROW.
 * DESIGN.md R7: the raw CV is compared with tau (the printed /sqrt(dim) bounds it < 1). */
adahop_pattern_t adahop_classify_cv(double cv_row, double cv_col, const adahop_params_t* p);

/* ------------------------------------------------------------- calibration (§5.1) */

/* Pattern statistics of a rows x cols tensor T (dt = BF16 or F32, leading dim ld):
 * row_stats[i*4 + {0,1,2,3}] = {sum x, sum x^2, sum |x|, max |x|} over row i (fp64),
 * col_stats[j*4 + ...]       = the same over column j (fp64).
 * Multi-rank callers sum-all-reduce col_stats[.,0..2] and max-all-reduce col_stats[.,3]
 * before adahop_classify. Workspace: adahop_stats_workspace_bytes(rows, cols). */
size_t adahop_stats_workspace_bytes(int64_t rows, int64_t cols);
adahop_status_t adahop_stats(const void* T, adahop_dtype_t dt, int64_t rows, int64_t cols,
                             int64_t ld, double* row_stats, double* col_stats, void* ws,
                             size_t ws_bytes, adahop_stream_t stream);

/* CV sums from statistics (App. A; population std). d_cv is a device array of 4:
 * d_cv[0] = sum_i std(T_i,:)/(mean|T_i,:| + eps) over the `rows` given rows (each has
 * `cols` elements); d_cv[1] = sum_j std(T_:,j)/(mean|T_:,j| + eps) over `cols` columns,
 * each with `col_count` elements (the global row count under token sharding);
 * d_cv[2] = CV_row = d_cv[0] / rows, d_cv[3] = CV_col = d_cv[1] / cols, and
 * d_pattern[0] = the App. A decision (R7) on them — the pattern of T on a
 * single rank. Multi-rank (token-sharded) calibration, all arithmetic in the library:
 *   adahop_stats -> all-reduce col_stats (SUM of [.,0..2], MAX of [.,3])
 *   -> adahop_classify(col_count = global rows) -> all-reduce d_cv[0] (SUM)
 *   -> adahop_classify_sums(rows_global) -> the global pattern, identical on every rank. */
adahop_status_t adahop_classify(const double* row_stats, int64_t rows, const double* col_stats,
                                int64_t cols, int64_t col_count, const adahop_params_t* p,
                                double* d_cv, uint8_t* d_pattern, adahop_stream_t stream);

/* The App. A decision from CV sums already reduced over all ranks: reads d_cv[0] (row-CV sum
 * over the rows_global rows of all ranks) and d_cv[1] (column-CV sum over `cols` columns), writes
 * d_cv[2] = d_cv[0] / rows_global, d_cv[3] = d_cv[1] / cols and d_pattern[0] (device). */
adahop_status_t adahop_classify_sums(double* d_cv, int64_t rows_global, int64_t cols, const adahop_params_t* p,
                                     uint8_t* d_pattern, adahop_stream_t stream);

/* One-call calibration of one tensor for one step on a single rank: stats + classify.
 * d_cv (4 doubles, as adahop_classify) and d_pattern (1 byte) are device outputs.
 * Workspace: adahop_calibrate_workspace_bytes(rows, cols). */
size_t adahop_calibrate_workspace_bytes(int64_t rows, int64_t cols);
adahop_status_t adahop_calibrate(const void* T, adahop_dtype_t dt, int64_t rows, int64_t cols,
                                 int64_t ld, const adahop_params_t* p, void* ws, size_t ws_bytes,
                                 double* d_cv, uint8_t* d_pattern, adahop_stream_t stream);

/* n calibration steps at once — the operands of one training step (§5.1: every linear's X, W and
 * G_Y) — in three kernel launches per 32 tensors instead of three per tensor. Tensor i
 * is T[i] (device, dtype dt for all) with rows[i] x cols[i] elements, row pitch ld[i] (host arrays
 * of n entries); results go to d_cv[4 i .. 4 i + 3] and d_pattern[i] exactly as n adahop_calibrate
 * calls would write them (same partition and reduction order: bitwise equal). The workspace is
 * the n single-tensor workspaces back to back (adahop_calibrate_batch_workspace_bytes). */
size_t adahop_calibrate_batch_workspace_bytes(int32_t n, const int64_t* rows, const int64_t* cols);
adahop_status_t adahop_calibrate_batch(int32_t n, const void* const* T, adahop_dtype_t dt, const int64_t* rows,
                                       const int64_t* cols, const int64_t* ld, const adahop_params_t* p, void* ws,
                                       size_t ws_bytes, double* d_cv, uint8_t* d_pattern, adahop_stream_t stream);

/* Outlier severity for a per-layer OE k (DESIGN R16, after App. D): called after
 * adahop_calibrate_batch with the same n / rows / cols / ws (it reads the row and column statistics
 * left there), writes d_counts[2 i] = the rows of tensor i whose max |x| exceeds kappa * mean |x|
 * (mean over all entries) and d_counts[2 i + 1] = the columns likewise (int32, device). One launch
 * per 32 tensors; kappa > 0 (the reading uses 32). */
adahop_status_t adahop_calibrate_batch_outliers(int32_t n, const int64_t* rows, const int64_t* cols, const void* ws,
                                                size_t ws_bytes, double kappa, int32_t* d_counts,
                                                adahop_stream_t stream);

/* ------------------------------------------------------------------- hot path */

/* Generic AdaHOP GEMM in stored form: C[M x N] = A_store[M x K] · B_store[N x K]^T under
 * `strategy`. A_store / B_store are views of bf16 memory:
 *   a_kstrided == 0: A_store[m][k] = A[m*lda + k]   (K contiguous)
 *   a_kstrided == 1: A_store[m][k] = A[k*lda + m]   (K strided: the transposing quant)
 * and likewise for B. C is written with leading dimension ldc in out_dt.
 * OE-Left extracts rows of A_store, OE-Right rows of B_store (= columns of B). */
size_t adahop_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, adahop_strategy_t s,
                                   const adahop_params_t* p);
adahop_status_t adahop_gemm(const void* A, int32_t a_kstrided, int64_t lda, const void* B,
                            int32_t b_kstrided, int64_t ldb, void* C, adahop_dtype_t out_dt,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, adahop_strategy_t s,
                            const adahop_params_t* p, void* ws, size_t ws_bytes,
                            adahop_stream_t stream);

/* Linear-layer paths. X: T x d_in, W: d_out x d_in, G_Y: T x d_out, all bf16
 * row-major and contiguous. Outputs contiguous in out_dt.
 *   fwd:   Y   = X W^T      (A_store = X,     B_store = W)      M=T,     N=d_out, K=d_in
 *   dgrad: G_X = G_Y W      (A_store = G_Y,   B_store = W^T)    M=T,     N=d_in,  K=d_out
 *   wgrad: G_W = G_Y^T X    (A_store = G_Y^T, B_store = X^T)    M=d_out, N=d_in,  K=T
 * wgrad additionally requires T % 32 == 0. Under token-row data parallelism each rank
 * calls wgrad on its shard and the caller all-reduces G_W (fp32) across ranks. */
size_t adahop_workspace_bytes(adahop_path_t path, int64_t T, int64_t d_in, int64_t d_out,
                              adahop_strategy_t s, const adahop_params_t* p);
adahop_status_t adahop_linear_fwd(const void* X, const void* W, void* Y, adahop_dtype_t out_dt,
                                  int64_t T, int64_t d_in, int64_t d_out, adahop_strategy_t s,
                                  const adahop_params_t* p, void* ws, size_t ws_bytes,
                                  adahop_stream_t stream);
adahop_status_t adahop_linear_dgrad(const void* GY, const void* W, void* GX, adahop_dtype_t out_dt,
                                    int64_t T, int64_t d_in, int64_t d_out, adahop_strategy_t s,
                                    const adahop_params_t* p, void* ws, size_t ws_bytes,
                                    adahop_stream_t stream);
adahop_status_t adahop_linear_wgrad(const void* GY, const void* X, void* GW, adahop_dtype_t out_dt,
                                    int64_t T, int64_t d_in, int64_t d_out, adahop_strategy_t s,
                                    const adahop_params_t* p, void* ws, size_t ws_bytes,
                                    adahop_stream_t stream);

/* One linear layer's three matmuls at once (fwd Y = X W^T, dgrad G_X = G_Y W, wgrad
 * G_W = G_Y^T X) with strategies s[0..2] = {fwd, dgrad, wgrad}. Same results as the
 * three calls above, but every input tensor is read once: a dual-orientation quantisation
 * pass emits both FP4 layouts of X (fwd A, wgrad B), W (fwd B, dgrad B) and G_Y (dgrad A,
 * wgrad A) — the quantised copies the paper keeps for backward. Requires T, d_in,
 * d_out multiples of 32. Outputs Y [T x d_out] and G_X [T x d_in] contiguous in out_dt,
 * G_W [d_out x d_in] contiguous in gw_dt (fp32 for the data-parallel all-reduce).
 * G_W is this rank's partial under token sharding (the caller all-reduces it).
 * With a wgrad OE-Right strategy (s[2], eq:oe_right P:280) and oe_k <= 64 the outlier product
 * A B_out = G_Y^T X[:, S] is accumulated inside G_Y's quantisation pass (transform,
 * quantisation and the outlier path in one kernel) instead of a separate BF16 GEMM; its fp32
 * partials are summed in a fixed order, so results are deterministic (run to run and graph vs
 * eager) and equal to the BF16-GEMM form to fp32 rounding of the outlier columns. */
size_t adahop_layer_workspace_bytes(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                    const adahop_params_t* p);
adahop_status_t adahop_linear_layer(const void* X, const void* W, const void* GY, void* Y, void* GX, void* GW,
                                    adahop_dtype_t out_dt, adahop_dtype_t gw_dt, int64_t T, int64_t d_in,
                                    int64_t d_out, const adahop_strategy_t* s, const adahop_params_t* p, void* ws,
                                    size_t ws_bytes, adahop_stream_t stream);

/* The same layer split into the two halves of a training step ("For activation tensors in
 * the Forward path, both the quantized residual and the BF16 outlier tensor are saved to the
 * context for backpropagation").
 *   adahop_linear_forward:  FOID + dual quantisation of X and W, Y = X W^T (fwd strategy s[0]);
 *                           writes the context `ctx` (caller-owned device memory of
 *                           adahop_linear_ctx_bytes, 256-byte aligned): the column-layout FP4
 *                           codes + E8M0 scales of X (wgrad B) and W (dgrad B), and the OE
 *                           indices + raw BF16 slices of their extracted columns.
 *   adahop_linear_backward: FOID + dual quantisation of G_Y, G_X = G_Y W and G_W = G_Y^T X from
 *                           the context. X (bf16, T x d_in) is read only when the wgrad's BF16
 *                           part multiplies by all of X — wgrad OE-Left (A_out B) or the
 *                           Lv2 BF16 wgrad; adahop_linear_backward_needs_x tells the
 *                           caller whether it must keep X alive (pass NULL otherwise).
 * Results are bitwise those of adahop_linear_layer with the same arguments (same kernels, same
 * inputs), except the k extracted rows of G_W (wgrad OE-Left) and of G_X (dgrad OE-Left): the layer
 * call accumulates those outlier products in a quant pass (X's / W's), the split backward, which has
 * neither pass, in a BF16 GEMM — two fp32 summation orders of the same products that agree to
 * rounding (DESIGN R15). The context must not be modified between the two calls; W must be unchanged. Both
 * calls use the workspace size adahop_linear_split_workspace_bytes (scratch, may be shared). */
size_t adahop_linear_ctx_bytes(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                               const adahop_params_t* p);
size_t adahop_linear_split_workspace_bytes(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                           const adahop_params_t* p);
int32_t adahop_linear_backward_needs_x(const adahop_strategy_t* s, const adahop_params_t* p);   /* host, pure */
adahop_status_t adahop_linear_forward(const void* X, const void* W, void* Y, adahop_dtype_t out_dt, int64_t T,
                                      int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                      const adahop_params_t* p, void* ctx, size_t ctx_bytes, void* ws,
                                      size_t ws_bytes, adahop_stream_t stream);
adahop_status_t adahop_linear_backward(const void* GY, const void* W, const void* X, void* GX, void* GW,
                                       adahop_dtype_t gx_dt, adahop_dtype_t gw_dt, int64_t T, int64_t d_in,
                                       int64_t d_out, const adahop_strategy_t* s, const adahop_params_t* p,
                                       const void* ctx, size_t ctx_bytes, void* ws, size_t ws_bytes,
                                       adahop_stream_t stream);

/* ------------------------------------------------------- debug / parity entry points */

/* Fused IHT + MXFP4 quantisation of a stored operand (the production kernels), with the
 * results converted to canonical layouts: codes_canon R x K/2 bytes (element 2j in the
 * low nibble), scales_canon R x K/32 bytes of biased E8M0 (e + 127). in is bf16 or f32:
 * k_strided == 0: row r = in[r*ld + 0..K); k_strided == 1: in[k*ld + r].
 * zero_rows (nzero sorted int32, device; may be NULL when nzero == 0) are masked to +0
 * before the transform (the OE residual). had_out (nullable, R x K f32) receives the
 * fp32 Hadamard output that enters the quantiser. */
adahop_status_t adahop_debug_iht_quant(const void* in, adahop_dtype_t dt, int64_t R, int64_t K,
                                       int64_t ld, int32_t k_strided, const int32_t* zero_rows,
                                       int32_t nzero, float* had_out, uint8_t* codes_canon,
                                       uint8_t* scales_canon, void* ws, size_t ws_bytes,
                                       adahop_stream_t stream);
size_t adahop_debug_workspace_bytes(int64_t R, int64_t K);

/* One-pass dual-orientation IHT + quantisation of a bf16 tensor T [R x C] (pitch ld elements):
 * the row operand (stored rows = R, K = C: q_row [R x C/2], scales_row [R x C/32]) and the
 * column operand (stored rows = C, K = R: q_col [C x R/2], scales_col [C x R/32]) — the two
 * layouts the three GEMMs of one linear need (eq:forward / eq:backward_gw / eq:backward_gx,
 * P:74-78; the quantised activations kept for backward). row_zero /
 * col_zero (sorted int32, device, <= 256 each) are the OE rows / columns: masked to zero blocks
 * and copied raw to slice_row [nrow_zero x C] / slice_col [ncol_zero x R] bf16 (nullable).
 * Canonical code / scale layouts as adahop_debug_iht_quant. R, C multiples of 32.
 * ws >= adahop_debug_workspace_bytes(R, C) + adahop_debug_workspace_bytes(C, R). */
adahop_status_t adahop_debug_quant_dual(const void* in, adahop_dtype_t dt, int64_t R, int64_t C, int64_t ld,
                                       const int32_t* row_zero, int32_t nrow_zero, const int32_t* col_zero,
                                       int32_t ncol_zero, uint8_t* q_row, uint8_t* scales_row, uint8_t* q_col,
                                       uint8_t* scales_col, void* slice_row, void* slice_col, void* ws,
                                       size_t ws_bytes, adahop_stream_t stream);

/* FOID: idx_sorted[0..min(k,R)) = ascending indices of the top-k stored rows by
 * the fp64 probe variance (ties -> lower index); keys_out (nullable) = the R keys. */
adahop_status_t adahop_debug_foid(const void* in, adahop_dtype_t dt, int64_t R, int64_t K,
                                  int64_t ld, int32_t k_strided, int32_t k, int32_t probe,
                                  int32_t* idx_sorted, double* keys_out, void* ws,
                                  size_t ws_bytes, adahop_stream_t stream);

/* Block-scaled MXFP4 GEMM on canonical operands: C[M x N] (f32 or bf16, ldc) =
 * deq(A codes/scales) · deq(B codes/scales)^T, using the production tcgen05 kernel. */
adahop_status_t adahop_debug_gemm_mxf4(const uint8_t* a_codes, const uint8_t* a_scales,
                                       const uint8_t* b_codes, const uint8_t* b_scales, void* C,
                                       adahop_dtype_t out_dt, int64_t ldc, int64_t M, int64_t N,
                                       int64_t K, void* ws, size_t ws_bytes,
                                       adahop_stream_t stream);
size_t adahop_debug_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);

/* The same GEMM kernel alone (one launch, no scale conversion): a_sf / b_sf are already in the
 * tcgen05 block-scaled layout the quantiser writes (adahop_debug_sf_bytes(rows, K) bytes each,
 * see DESIGN.md §5). Used to time the GEMM kernel by itself (bench.py's library comparison). */
size_t adahop_debug_sf_bytes(int64_t rows, int64_t K);
adahop_status_t adahop_debug_gemm_mxf4_tcsf(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes,
                                            const uint8_t* b_sf, void* C, adahop_dtype_t out_dt, int64_t ldc,
                                            int64_t M, int64_t N, int64_t K, adahop_stream_t stream);

/* E2M1 element conversion used by the quantiser (hardware cvt.rn.satfinite.e2m1x2) and
 * its software statement (nearest of {0,.5,1,1.5,2,3,4,6}, ties to even mantissa,
 * saturating, sign = signbit): one code per input (device arrays of n). */
adahop_status_t adahop_debug_e2m1(const float* v, int64_t n, uint8_t* codes_hw, uint8_t* codes_sw,
                                  adahop_stream_t stream);
/* Compare the two conversions on every finite fp32 bit pattern in [lo, hi) (hi <= 2^32);
 * adds the mismatch count to *d_mismatches and atomically min-reduces the first bad
 * pattern into *d_first_bad (both device, caller-initialised). */
adahop_status_t adahop_debug_e2m1_exhaustive(uint64_t lo, uint64_t hi,
                                             unsigned long long* d_mismatches,
                                             uint32_t* d_first_bad, adahop_stream_t stream);

/* Number of kernel launches the last successful hot-path call on this thread issued
 * (host counter; used by bench.py to report gpu_launches). */
int32_t adahop_last_launch_count(void);

/* Optional stage timing (tab:latency breakdown): `events` is a host array of 5
 * cudaEvent_t (or NULL to disable) used by the following hot-path calls on this thread:
 * [0] start, [1] after FOID, [2] after IHT+quant of both operands (with the OE-slice gathers and,
 * in the layer / backward calls, the fused wgrad OE-Right outlier product), [3] after the
 * remaining BF16 outlier GEMMs + split-K folds, [4] after the MXFP4 GEMMs, whose epilogues write
 * the outlier entries (the fused scatter) — or after the Lv2 BF16 GEMM. */
void adahop_set_stage_events(void* events);

#ifdef __cplusplus
}
#endif
#endif /* ADAHOP_H_ */
