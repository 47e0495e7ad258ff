// kernels.h — host-side launchers of the AdaHOP sm_100a kernels (internal to libadahop).
#pragma once
#include "epilogue.cuh"
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace adahop {

// ------------------------------------------------------------------ host-side knobs and caches
// Experiment knobs: read from the environment only in experiment builds (build.py --define
// ADAHOP_EXPERIMENTS=1, used by scripts/micro); the product library always uses the defaults.
#ifndef ADAHOP_EXPERIMENTS
#define ADAHOP_EXPERIMENTS 0
#endif
inline int knob(const char* name, int dflt) {
#if ADAHOP_EXPERIMENTS
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

// Per-device one-time setup. cudaFuncSetAttribute (and occupancy queries) apply to the device
// that is current at the call, so the "done" record is kept per device ordinal (bit d of the
// mask). Concurrent first calls may both run `fn`, which must be idempotent; the mask itself is
// atomic, so the library stays thread-safe (include/adahop.h).
int current_device();
template <typename Fn>
inline cudaError_t once_per_device(std::atomic<uint64_t>& done, Fn&& fn) {
  const int dev = current_device();
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  const uint64_t bit = uint64_t(1) << dev;
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = fn();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}
// A per-device cached positive integer (0 = not computed yet).
struct PerDeviceInt {
  std::atomic<int> v[64];
  PerDeviceInt() { for (auto& x : v) x.store(0); }
};

// Kernel launch with programmatic dependent launch (PDL) on the stream, optionally as 2-CTA
// clusters. (Experiment builds: ADAHOP_PDL=0 launches without the PDL attribute.)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster_x > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = unsigned(cluster_x);
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = na ? at : nullptr;
  cfg.numAttrs = unsigned(na);
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// quant.cu
// zero_rows (sorted, nzero) are the OE rows: masked to +0 in the residual and, when
// slice != nullptr, copied raw (bf16) into slice[slot][0..K) — the outlier gather is fused.
cudaError_t launch_iht_quant(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld,
                             int kstrided, const int32_t* zero_rows, int nzero, uint8_t* codes,
                             uint8_t* sf, float* had_out, __nv_bfloat16* slice, bool sw_cvt,
                             int num_sms, cudaStream_t st);
// One pass over bf16 T [R x C] (pitch ld): row quantisation (rows, K = C) and column
// quantisation (columns, K = R), each with its own OE mask / slice (nullable).
cudaError_t launch_iht_quant_dual(const __nv_bfloat16* in, int64_t R, int64_t C, int64_t ld,
                                  const int32_t* row_zero, int nrow_zero, __nv_bfloat16* slice_row,
                                  uint8_t* q_row, uint8_t* sf_row, const int32_t* col_zero, int ncol_zero,
                                  __nv_bfloat16* slice_col, uint8_t* q_col, uint8_t* sf_col, int num_sms,
                                  cudaStream_t st);
bool dual_quant_supported(int64_t R, int64_t C, bool row_mask, bool col_mask);
// quant_tc.cu — Hadamard on the tensor cores, quantisation in the epilogue (bf16 sources).
bool quant_use_tc();   // experiment builds: ADAHOP_QUANT_SCALAR=1 selects the butterfly kernels
int quant_last_launches();   // kernels launched by the last launch_iht_quant / launch_iht_quant_dual
bool quant_tc_supported(int64_t R, int64_t C, int64_t ld, const void* in, bool row_mask, bool col_mask);
struct QuantTcJob {
  const __nv_bfloat16* in; int64_t R, C, ld;
  const int32_t* row_zero; int nrow_zero; __nv_bfloat16* slice_row; uint8_t* q_row; uint8_t* sf_row; float* had_row;
  const int32_t* col_zero; int ncol_zero; __nv_bfloat16* slice_col; uint8_t* q_col; uint8_t* sf_col; float* had_col;
  // optional fused outlier product of this tensor (the wgrad's, eq:oe_right P:280 / eq:oe_left P:273):
  // P[j][c] = sum_r T[r][c] or_slice[j][r] for j < or_kk (<= 64), c < C, left as per-(band, CTA)
  // partials in or_part (quant_tc_or_part_bytes bytes) that quant_tc_or_patch describes to the
  // MXFP4 GEMM epilogue; or_slice [or_kk][R] bf16 must be complete before the launch
  const __nv_bfloat16* or_slice = nullptr; int or_kk = 0; float* or_part = nullptr; size_t or_part_bytes = 0;
  unsigned* or_ticket = nullptr;   // 4 bytes, zeroed by the launch, counted by the GEMM pre-fold
};
// Up to 3 tensors in one persistent launch (same orientation set for all), up to two of them with
// a fused outlier product (their or_slice complete before the launch).
// OE slices are produced by a separate gather launch; *launches (nullable) counts every launch.
// or_fused (nullable, n entries, indexed like jobs) tells whether a job's outlier product was
// computed (else the caller runs the BF16 outlier GEMM: the products are fused only on the
// dual-orientation kernel when they fit).
cudaError_t launch_quant_tc_multi(const QuantTcJob* jobs, int n, int num_sms, cudaStream_t st, int* launches,
                                  bool* or_fused);
size_t quant_tc_or_part_bytes(int64_t R, int64_t C, int kk, int num_sms);
OePatch quant_tc_or_patch(int64_t R, int64_t C, int kk, int num_sms, const float* part, unsigned* ticket, float* Dt,
                          const int32_t* idx, int mode);
cudaError_t launch_quant_tc(const __nv_bfloat16* in, int64_t R, int64_t C, int64_t ld, const int32_t* row_zero,
                            int nrow_zero, __nv_bfloat16* slice_row, uint8_t* q_row, uint8_t* sf_row, float* had_row,
                            const int32_t* col_zero, int ncol_zero, __nv_bfloat16* slice_col, uint8_t* q_col,
                            uint8_t* sf_col, float* had_col, int num_sms, cudaStream_t st);
cudaError_t launch_sf_convert(const uint8_t* src, int64_t R, int64_t K, uint8_t* dst,
                              bool to_canonical, cudaStream_t st);
// FOID: probe keys + top-k -> idx_sorted[min(k,R)] (ascending). `keys` points to a scratch
// buffer of foid_ws_bytes(R) bytes whose first R doubles receive the keys. R <= kFoidMaxRows:
// 16 select blocks of 4096 rows whose k <= 256 survivors the last block merges in 4096 slots.
constexpr int64_t kFoidMaxRows = 65536;
size_t foid_ws_bytes(int64_t R);
cudaError_t launch_foid(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld,
                        int kstrided, int k, int probe, double* keys, int32_t* idx_sorted,
                        cudaStream_t st);
cudaError_t launch_foid_keys_only(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld, int kstrided,
                                  int probe, double* keys, cudaStream_t st);
int foid_launches(int64_t R, int64_t K, int probe);
// Several FOIDs in two launches (keys, select); each job has its own foid_ws_bytes(R) scratch.
constexpr int kFoidMaxJobs = 6;
struct FoidJob {
  const void* in; int64_t R, K, ld; int kstrided, k, probe; double* scratch; int32_t* idx;
};
cudaError_t launch_foid_batch(const FoidJob* jobs, int n, bool in_f32, cudaStream_t st);
size_t stats_ws_bytes(int64_t R, int64_t C);   // workspace of launch_stats (bytes)
// one calibration step of one tensor: stats, CV partials, classification (3 launches)
size_t calib_cvpart_bytes(int64_t R, int64_t C);
cudaError_t launch_calibrate(const void* in, bool in_f32, int64_t R, int64_t C, int64_t ld, double* rs, double* cs,
                             double* part, double* cvpart, double eps, double tau, double* d_cv, uint8_t* pattern,
                             cudaStream_t st);
// Several calibration steps (stats -> CV partials -> R/C/N) in three launches; every job uses
// the single-tensor workspace layout (rs, cs, stats partials `part`, cvpart) and gets the same
// bits as launch_calibrate.
constexpr int kCalibMaxJobs = 32;
struct CalibJob {
  const void* in; int64_t R, C, ld;
  double *rs, *cs, *part, *cvpart, *d_cv;
  uint8_t* pattern;
};
cudaError_t launch_calibrate_batch(const CalibJob* jobs, int n, bool in_f32, double eps, double tau, cudaStream_t st);
// counts[2 i], counts[2 i + 1] = the outlier rows / columns of job i (DESIGN R16) from the
// statistics launch_calibrate_batch left in jobs[i].rs / .cs
cudaError_t launch_outlier_counts_batch(const CalibJob* jobs, int n, double kappa, int32_t* counts, cudaStream_t st);
cudaError_t launch_stats(const void* in, bool in_f32, int64_t R, int64_t C, int64_t ld,
                         double* rs, double* cs, double* part, cudaStream_t st);
cudaError_t launch_classify_sums(double* d_cv, int64_t rows, int64_t cols, double tau, uint8_t* pattern,
                                 cudaStream_t st);
cudaError_t launch_classify(const double* rs, int64_t rows, int64_t row_len, const double* cs,
                            int64_t cols, int64_t col_len, double eps, double tau, double* d_cv,
                            uint8_t* pattern, cudaStream_t st);

cudaError_t launch_e2m1_codes(const float* v, int64_t n, uint8_t* hw, uint8_t* sw, cudaStream_t st);
cudaError_t launch_e2m1_exhaustive(uint64_t lo, uint64_t hi, unsigned long long* mism,
                                   unsigned int* first_bad, cudaStream_t st);

// gemm_mxf4.cu — C[M x N] = deq(A) deq(B)^T, A/B MXFP4 K-major (codes + tcgen05 SF layout)
struct Mxf4GemmArgs {
  const uint8_t* a_codes;
  const uint8_t* a_sf;
  const uint8_t* b_codes;
  const uint8_t* b_sf;
  void* C;
  bool out_f32;
  int64_t ldc, M, N, K;
  OePatch oe;   // outlier entries written by the epilogue (oe.mode 0: none)
};
cudaError_t launch_gemm_mxf4(const Mxf4GemmArgs& a, int num_sms, cudaStream_t st);
// gemm_mxf4_2sm.cu — CTA-pair (cta_group::2) version; variant = 128 (256x128 tiles, double-
// buffered accumulators) or 256 (256x256 tiles, single accumulator).
cudaError_t launch_gemm_mxf4_2sm(const Mxf4GemmArgs& a, int num_sms, int variant, cudaStream_t st);
// 2..3 MXFP4 GEMMs (the paths of one linear) in one persistent launch, clusters split by work
cudaError_t launch_gemm_mxf4_2sm_group(const Mxf4GemmArgs* a, int n, int num_sms, cudaStream_t st, bool* launched);
// split-K over clusters of `split` CTA pairs for long-K GEMMs with few output tiles
cudaError_t launch_gemm_mxf4_2sm_split(const Mxf4GemmArgs& a, int num_sms, int split, cudaStream_t st,
                                       bool* launched);

// gemm_bf16.cu — D[Mb x Nb] = A[Mb x K] B[Nb x K]^T in BF16 (fp32 accumulate).
// A/B are K-major (a_mn = 0: A[m*lda + k]) or MN-major (a_mn = 1: A[k*lda + m]).
// mode 0: D written densely to C (out dtype, ldc); mode 1: fp32 split-K partials to
// part[split][Mb][npad] (npad = padded Nb), reduced afterwards by launch_outlier_reduce.
struct Bf16GemmArgs {
  const __nv_bfloat16* A;
  int a_mn;
  int64_t lda;
  const __nv_bfloat16* B;
  int b_mn;
  int64_t ldb;
  int64_t Mb, Nb, K;
  int mode;
  void* C;
  bool out_f32;
  int64_t ldc;
  float* part;
  int splits;
  int64_t npad;
  float* Dt = nullptr;   // mode 1 with splits == 1: the transposed product Dt[j][m] written directly (no fold)
};
// the full BF16 product (mode 0) on CTA pairs; *launched = false: use launch_gemm_bf16
cudaError_t launch_gemm_bf16_2sm(const Bf16GemmArgs& a, int num_sms, cudaStream_t st, bool* launched);

int64_t bf16_gemm_npad(int64_t Nb);
int bf16_gemm_splits(int64_t Mb, int64_t K, int num_sms);
cudaError_t launch_gemm_bf16(const Bf16GemmArgs& a, cudaStream_t st);
// Scatter-add of the outlier product into C (fused "scatter-add" stage):
// val(m, j) = sum_split part[split][m][j] (fixed order);
// scatter_cols (OE-Right): C[m][idx[j]] = val;  else (OE-Left): C[idx[j]][m] = val.
// The MXFP4 product is exactly 0 at those positions (disjoint support), so the store
// equals the add.
// Dt[j][m] = sum over the split-K partials (fixed order) of the outlier product D[m][j].
cudaError_t launch_outlier_fold(const float* part, int splits, int64_t Mb, int64_t npad, int k, float* Dt,
                                cudaStream_t st);

// tensor maps (api.cu)
bool make_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner,
                  uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                  CUtensorMapSwizzle swz);

}  // namespace adahop
