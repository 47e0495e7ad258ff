// api.cu — the C ABI of libadahop (include/adahop.h): validation, strategy dispatch,
// workspace carving and kernel sequencing. No allocation, no host sync on the hot path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <initializer_list>
#include <mutex>

#include "../../include/adahop.h"
#include "common.cuh"
#include "kernels.h"

using namespace adahop;

namespace {

thread_local int32_t g_launches = 0;
thread_local cudaEvent_t* g_stage_events = nullptr;  // optional per-stage timing (bench)

inline void stage_mark(int i, cudaStream_t st) {
  if (!g_stage_events) return;
  // inside CUDA-graph capture an "external" record node keeps the event observable
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  if (cap == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(g_stage_events[i], st, cudaEventRecordExternal);
  else
    cudaEventRecord(g_stage_events[i], st);
}

// ---------------------------------------------------------------------- driver / device
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct DevInfo {
  int sms = 0;
  int major = 0;
  bool ok = false;
};
DevInfo dev_info() {
  static DevInfo cache[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DevInfo{};
  std::lock_guard<std::mutex> lk(mu);
  if (!cache[dev].ok) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return DevInfo{};
    cache[dev].sms = prop.multiProcessorCount;
    cache[dev].major = prop.major;
    cache[dev].ok = true;
  }
  return cache[dev];
}

adahop_status_t check_device(DevInfo* out) {
  DevInfo d = dev_info();
  if (!d.ok || d.major != 10) return ADAHOP_E_NO_DEVICE;
  if (!encode_fn()) return ADAHOP_E_CUDA;
  if (out) *out = d;
  return ADAHOP_OK;
}

#define ADAHOP_LAUNCH(expr)                                 \
  do {                                                      \
    cudaError_t e_ = (expr);                                \
    if (e_ != cudaSuccess) return ADAHOP_E_CUDA;            \
  } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// MXFP4 GEMM kernel choice: ADAHOP_GEMM_VARIANT = 1 (1-CTA 128x128), 128 or 256 (CTA pairs).
int gemm_variant() {
  static const int v = knob("ADAHOP_GEMM_VARIANT", 256);
  return v;
}
// ADAHOP_GEMM_SPLITK (experiment builds): 0 = 256x128 tiles instead of split-K clusters,
// 2 / 4 = that many pairs per cluster whenever the split applies
int gemm_splitk() {
  static const int v = knob("ADAHOP_GEMM_SPLITK", 1);
  return v;
}

// allow_splitk = false (the layer and split-step calls): one accumulation order per output for
// every schedule, so that the split forward / backward stays bitwise equal to the layer call
// whether or not either call groups its GEMMs (§6.4); those calls group a starving wgrad instead.
cudaError_t run_gemm_mxf4(const Mxf4GemmArgs& a, int sms, cudaStream_t st, bool allow_splitk = true) {
  int v = gemm_variant();
  if (v == 1 || a.M <= 128) return launch_gemm_mxf4(a, sms, st);
  // long-K GEMMs with fewer 256x256 tiles than half the CTA pairs (e.g. the Llama-3.2-1B k/v
  // wgrad, 512 x 2048, K = 16384): the 256x128 double-buffered tiles keep twice as many pairs
  // busy (27 -> 22 us measured)
  const int64_t tiles256 = ((a.M + 255) / 256) * ((a.N + 255) / 256);
  if (v == 256 && a.K >= 8192 && 2 * tiles256 < sms / 2) {
    // split-K over clusters of 4 (or 2) pairs, one 256x256 tile per cluster, partials summed in
    // distributed shared memory (e.g. 16 tiles x 4 pairs: 64 of the 74 pairs busy)
    const int force = gemm_splitk();
    if (force != 0 && allow_splitk)
      for (int split = 4; split >= 2; split /= 2) {
        if (force > 1 ? split != force : split * tiles256 > sms / 2) continue;
        bool launched = false;
        const cudaError_t e = launch_gemm_mxf4_2sm_split(a, sms, split, st, &launched);
        if (e != cudaSuccess || launched) return e;
      }
    v = 128;
  }
  return launch_gemm_mxf4_2sm(a, sms, v, st);
}

// Grouped launch of a linear's MXFP4 GEMMs when their total work is small (<= 0.8 TFLOP) and the
// launcher's rule accepts it (one problem starving the machine; launch_gemm_mxf4_2sm_group).
// Experiment builds: ADAHOP_GEMM_GROUP = 0 never, 2 = any size.
bool group_gemms(double flops) {
  static const int v = knob("ADAHOP_GEMM_GROUP", 1);
  return v == 2 || (v == 1 && flops <= 0.8e12);
}

// The full BF16 product (Lv2 CC): CTA pairs with 256 x 256 tiles, else the 1-CTA kernel.
cudaError_t run_gemm_bf16_full(const Bf16GemmArgs& a, int sms, cudaStream_t st) {
  bool launched = false;
  const cudaError_t e = launch_gemm_bf16_2sm(a, sms, st, &launched);
  if (e != cudaSuccess || launched) return e;
  return launch_gemm_bf16(a, st);
}

// ---------------------------------------------------------------------- workspace carving
struct Carver {
  size_t off = 0;
  size_t take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    const size_t at = off;
    off += bytes;
    return at;
  }
};

struct GemmPlan {
  int kk = 0;               // extracted rows (0 = no OE)
  int64_t rows_oe = 0;      // rows of the OE operand
  int64_t mbig = 0;         // rows of the big operand of the outlier GEMM
  int64_t npad = 0;
  int splits = 1;
  size_t qa_codes = 0, qa_sf = 0, qb_codes = 0, qb_sf = 0;
  size_t keys = 0, idx = 0, slice = 0, part = 0, dt = 0;
  size_t total = 0;
};

bool plan_gemm(int64_t M, int64_t N, int64_t K, adahop_strategy_t s, const adahop_params_t* p,
               int num_sms, GemmPlan* g) {
  Carver c;
  *g = GemmPlan{};
  if (s == ADAHOP_BF16) {
    g->total = 256;
    return true;
  }
  g->qa_codes = c.take(size_t(M) * size_t(K / 2));
  g->qa_sf = c.take(size_t(sf_bytes(M, K)));
  g->qb_codes = c.take(size_t(N) * size_t(K / 2));
  g->qb_sf = c.take(size_t(sf_bytes(N, K)));
  const bool oe = (s == ADAHOP_OE_LEFT_IHT || s == ADAHOP_OE_RIGHT_IHT) && p->oe_k > 0;
  if (oe) {
    g->rows_oe = s == ADAHOP_OE_LEFT_IHT ? M : N;
    g->mbig = s == ADAHOP_OE_LEFT_IHT ? N : M;
    g->kk = int(std::min<int64_t>(p->oe_k, g->rows_oe));
    g->keys = c.take(foid_ws_bytes(g->rows_oe));
    g->idx = c.take(size_t(g->kk) * 4);
    g->slice = c.take(size_t(g->kk) * size_t(K) * 2);
    g->npad = bf16_gemm_npad(g->kk);
    g->splits = bf16_gemm_splits(g->mbig, K, num_sms);
    g->part = c.take(size_t(g->splits) * size_t(g->mbig) * size_t(g->npad) * 4);
    g->dt = c.take(size_t(g->kk) * size_t(g->mbig) * 4);
  }
  g->total = c.take(0) + 256;
  return true;
}

adahop_status_t validate_params(const adahop_params_t* p) {
  if (!p) return ADAHOP_E_INVALID_ARG;
  if (p->had_block != 32) return ADAHOP_E_UNSUPPORTED;
  if (p->oe_k < 0 || p->foid_probe < 1 || (p->level != 1 && p->level != 2))
    return ADAHOP_E_INVALID_ARG;
  if (p->oe_k > 256) return ADAHOP_E_UNSUPPORTED;
  return ADAHOP_OK;
}

}  // namespace

// ============================================================================ PDL switch
namespace adahop {
int current_device() {
  int d = -1;
  return cudaGetDevice(&d) == cudaSuccess && d >= 0 && d < 64 ? d : -1;
}

// ADAHOP_OR_FUSED=0 (experiment builds) runs the wgrad OE-Right product as a BF16 GEMM instead
bool or_fusion_enabled() {
  static const int v = knob("ADAHOP_OR_FUSED", 1);
  static const bool on = v == 1 || v == 3 || v == 4;
  return on;
}

// ADAHOP_OR_FUSED=4 (experiment builds): only the OE-Right product is fused
bool or_left_enabled() {
  static const bool on = knob("ADAHOP_OR_FUSED", 1) != 4;
  return on;
}

// ADAHOP_OR_DGRAD=0 (experiment builds): the dgrad's OE-Left product as a BF16 GEMM
bool or_dgrad_enabled() {
  static const bool on = knob("ADAHOP_OR_DGRAD", 1) != 0;
  return on;
}

bool pdl_enabled() {
  static const bool on = knob("ADAHOP_PDL", 1) != 0;
  return on;
}
}  // namespace adahop

// ============================================================================ tensor maps
namespace adahop {
bool make_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner,
                  uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                  CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
}  // namespace adahop

// ============================================================================ C ABI
extern "C" {

void adahop_default_params(adahop_params_t* p) {
  if (!p) return;
  p->had_block = 32;
  p->oe_k = 64;
  p->foid_probe = 64;
  p->level = 1;
  p->tau = 2.0f;
  p->eps = 1e-8f;
}

int32_t adahop_abi_version(void) { return ADAHOP_ABI_VERSION; }

int32_t adahop_last_launch_count(void) { return g_launches; }

void adahop_set_stage_events(void* events) { g_stage_events = static_cast<cudaEvent_t*>(events); }

const char* adahop_status_string(adahop_status_t s) {
  switch (s) {
    case ADAHOP_OK: return "ok";
    case ADAHOP_E_INVALID_ARG: return "invalid argument";
    case ADAHOP_E_SHAPE: return "shape error";
    case ADAHOP_E_UNSUPPORTED: return "unsupported configuration";
    case ADAHOP_E_WORKSPACE: return "workspace too small or misaligned";
    case ADAHOP_E_CUDA: return "CUDA error";
    case ADAHOP_E_NO_DEVICE: return "no sm_100 device";
  }
  return "unknown status";
}

adahop_strategy_t adahop_strategy_for_pair(adahop_pattern_t l, adahop_pattern_t r, int32_t level) {
  const bool R_ = l == ADAHOP_PAT_ROW, lC = l == ADAHOP_PAT_COL, lN = l == ADAHOP_PAT_NONE;
  const bool rR = r == ADAHOP_PAT_ROW, rC = r == ADAHOP_PAT_COL, rN = r == ADAHOP_PAT_NONE;
  if (lC && rC) return level == 2 ? ADAHOP_BF16 : ADAHOP_OE_RIGHT_IHT;
  if (R_ && (rN || rR)) return ADAHOP_OE_LEFT_IHT;                      // RN, RR
  if ((R_ || lN) && rC) return ADAHOP_OE_RIGHT_IHT;                     // RC, NC
  return ADAHOP_IHT;                                                    // CN, NN, CR, NR
}

adahop_pattern_t adahop_majority_vote(const int32_t* per_step, int32_t n) {
  if (!per_step || n <= 0) return ADAHOP_PAT_INVALID;
  int cnt[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) {
    if (per_step[i] < 0 || per_step[i] > 2) return ADAHOP_PAT_INVALID;
    cnt[per_step[i]]++;
  }
  const int best = std::max(cnt[0], std::max(cnt[1], cnt[2]));
  if (cnt[ADAHOP_PAT_ROW] == best) return ADAHOP_PAT_ROW;
  if (cnt[ADAHOP_PAT_COL] == best) return ADAHOP_PAT_COL;
  return ADAHOP_PAT_NONE;
}

int32_t adahop_layer_strategies(adahop_pattern_t pat_x, adahop_pattern_t pat_w, adahop_pattern_t pat_gy,
                                int32_t level, adahop_strategy_t* out, adahop_pattern_t* fed_pairs) {
  auto ok = [](adahop_pattern_t q) { return q == ADAHOP_PAT_NONE || q == ADAHOP_PAT_ROW || q == ADAHOP_PAT_COL; };
  if (!out || !ok(pat_x) || !ok(pat_w) || !ok(pat_gy) || (level != 1 && level != 2)) return -1;
  auto tr = [](adahop_pattern_t q) {   // pattern of the transpose (R8)
    return q == ADAHOP_PAT_ROW ? ADAHOP_PAT_COL : (q == ADAHOP_PAT_COL ? ADAHOP_PAT_ROW : ADAHOP_PAT_NONE);
  };
  // fed pairs: fwd (X, W^T), dgrad (G_Y, W), wgrad (G_Y^T, X)
  const adahop_pattern_t fed[3][2] = {{pat_x, tr(pat_w)}, {pat_gy, pat_w}, {tr(pat_gy), pat_x}};
  for (int path = 0; path < 3; ++path) {
    out[path] = adahop_strategy_for_pair(fed[path][0], fed[path][1], level);
    if (fed_pairs) {
      fed_pairs[2 * path] = fed[path][0];
      fed_pairs[2 * path + 1] = fed[path][1];
    }
  }
  return 0;
}

adahop_pattern_t adahop_classify_cv(double cv_row, double cv_col, const adahop_params_t* p) {
  const double tau = p ? p->tau : 2.0;
  const bool row_hit = cv_col > tau, col_hit = cv_row > tau;
  if (row_hit && (!col_hit || cv_col >= cv_row)) return ADAHOP_PAT_ROW;
  if (col_hit) return ADAHOP_PAT_COL;
  return ADAHOP_PAT_NONE;
}

// ------------------------------------------------------------------------ calibration
size_t adahop_stats_workspace_bytes(int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return 0;
  return stats_ws_bytes(rows, cols);
}

adahop_status_t adahop_stats(const void* T, adahop_dtype_t dt, int64_t rows, int64_t cols,
                             int64_t ld, double* row_stats, double* col_stats, void* ws,
                             size_t ws_bytes, adahop_stream_t stream) {
  if (!T || !row_stats || !col_stats || !ws) return ADAHOP_E_INVALID_ARG;
  if (dt != ADAHOP_DT_BF16 && dt != ADAHOP_DT_F32) return ADAHOP_E_INVALID_ARG;
  if (rows <= 0 || cols <= 0 || ld < cols) return ADAHOP_E_SHAPE;
  if (ws_bytes < adahop_stats_workspace_bytes(rows, cols) || (reinterpret_cast<uintptr_t>(ws) & 255))
    return ADAHOP_E_WORKSPACE;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  g_launches = 0;
  ADAHOP_LAUNCH(launch_stats(T, dt == ADAHOP_DT_F32, rows, cols, ld, row_stats, col_stats,
                             static_cast<double*>(ws), reinterpret_cast<cudaStream_t>(stream)));
  g_launches = 2;
  return ADAHOP_OK;
}

adahop_status_t adahop_classify(const double* row_stats, int64_t rows, const double* col_stats,
                                int64_t cols, int64_t col_count, const adahop_params_t* p,
                                double* d_cv, uint8_t* d_pattern, adahop_stream_t stream) {
  if (!row_stats || !col_stats || !d_cv || !d_pattern || !p) return ADAHOP_E_INVALID_ARG;
  if (rows <= 0 || cols <= 0 || col_count <= 0) return ADAHOP_E_SHAPE;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  ADAHOP_LAUNCH(launch_classify(row_stats, rows, cols, col_stats, cols, col_count, double(p->eps),
                                double(p->tau), d_cv, d_pattern,
                                reinterpret_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return ADAHOP_OK;
}

adahop_status_t adahop_classify_sums(double* d_cv, int64_t rows_global, int64_t cols, const adahop_params_t* p,
                                     uint8_t* d_pattern, adahop_stream_t stream) {
  if (!d_cv || !d_pattern || !p) return ADAHOP_E_INVALID_ARG;
  if (rows_global <= 0 || cols <= 0) return ADAHOP_E_SHAPE;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  ADAHOP_LAUNCH(launch_classify_sums(d_cv, rows_global, cols, double(p->tau), d_pattern,
                                     reinterpret_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return ADAHOP_OK;
}

size_t adahop_calibrate_workspace_bytes(int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return 0;
  Carver c;
  c.take(size_t(rows) * 32);
  c.take(size_t(cols) * 32);
  c.take(adahop_stats_workspace_bytes(rows, cols));
  c.take(calib_cvpart_bytes(rows, cols));
  return c.take(0) + 256;
}

adahop_status_t adahop_calibrate(const void* T, adahop_dtype_t dt, int64_t rows, int64_t cols,
                                 int64_t ld, const adahop_params_t* p, void* ws, size_t ws_bytes,
                                 double* d_cv, uint8_t* d_pattern, adahop_stream_t stream) {
  if (!T || !p || !ws || !d_cv || !d_pattern) return ADAHOP_E_INVALID_ARG;
  if (rows <= 0 || cols <= 0 || ld < cols) return ADAHOP_E_SHAPE;
  if (ws_bytes < adahop_calibrate_workspace_bytes(rows, cols) ||
      (reinterpret_cast<uintptr_t>(ws) & 255))
    return ADAHOP_E_WORKSPACE;
  Carver c;
  uint8_t* base = static_cast<uint8_t*>(ws);
  double* rs = reinterpret_cast<double*>(base + c.take(size_t(rows) * 32));
  double* cs = reinterpret_cast<double*>(base + c.take(size_t(cols) * 32));
  const size_t sw = adahop_stats_workspace_bytes(rows, cols);
  double* sws = reinterpret_cast<double*>(base + c.take(sw));
  double* cvpart = reinterpret_cast<double*>(base + c.take(calib_cvpart_bytes(rows, cols)));
  if (dt != ADAHOP_DT_BF16 && dt != ADAHOP_DT_F32) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  ADAHOP_LAUNCH(launch_calibrate(T, dt == ADAHOP_DT_F32, rows, cols, ld, rs, cs, sws, cvpart, double(p->eps),
                                 double(p->tau), d_cv, d_pattern, reinterpret_cast<cudaStream_t>(stream)));
  g_launches = 3;
  return ADAHOP_OK;
}

size_t adahop_calibrate_batch_workspace_bytes(int32_t n, const int64_t* rows, const int64_t* cols) {
  if (n <= 0 || !rows || !cols) return 0;
  size_t total = 0;
  for (int32_t i = 0; i < n; ++i) {
    const size_t b = adahop_calibrate_workspace_bytes(rows[i], cols[i]);
    if (b == 0) return 0;
    total += (b + 255) & ~size_t(255);
  }
  return total;
}

adahop_status_t adahop_calibrate_batch(int32_t n, const void* const* T, adahop_dtype_t dt, const int64_t* rows,
                                       const int64_t* cols, const int64_t* ld, const adahop_params_t* p, void* ws,
                                       size_t ws_bytes, double* d_cv, uint8_t* d_pattern, adahop_stream_t stream) {
  if (n <= 0 || !T || !rows || !cols || !ld || !p || !ws || !d_cv || !d_pattern) return ADAHOP_E_INVALID_ARG;
  if (dt != ADAHOP_DT_BF16 && dt != ADAHOP_DT_F32) return ADAHOP_E_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i) {
    if (!T[i]) return ADAHOP_E_INVALID_ARG;
    if (rows[i] <= 0 || cols[i] <= 0 || ld[i] < cols[i]) return ADAHOP_E_SHAPE;
  }
  if (ws_bytes < adahop_calibrate_batch_workspace_bytes(n, rows, cols) || (reinterpret_cast<uintptr_t>(ws) & 255))
    return ADAHOP_E_WORKSPACE;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  int32_t launches = 0;
  for (int32_t i0 = 0; i0 < n; i0 += kCalibMaxJobs) {
    CalibJob jobs[kCalibMaxJobs];
    const int m = int(std::min<int32_t>(kCalibMaxJobs, n - i0));
    for (int k = 0; k < m; ++k) {
      const int32_t i = i0 + k;
      Carver c;   // the single-tensor layout of adahop_calibrate
      double* rs = reinterpret_cast<double*>(base + c.take(size_t(rows[i]) * 32));
      double* csum = reinterpret_cast<double*>(base + c.take(size_t(cols[i]) * 32));
      double* sws = reinterpret_cast<double*>(base + c.take(adahop_stats_workspace_bytes(rows[i], cols[i])));
      double* cvpart = reinterpret_cast<double*>(base + c.take(calib_cvpart_bytes(rows[i], cols[i])));
      jobs[k] = CalibJob{T[i], rows[i], cols[i], ld[i], rs, csum, sws, cvpart, d_cv + 4 * int64_t(i), d_pattern + i};
      base += (adahop_calibrate_workspace_bytes(rows[i], cols[i]) + 255) & ~size_t(255);
    }
    ADAHOP_LAUNCH(launch_calibrate_batch(jobs, m, dt == ADAHOP_DT_F32, double(p->eps), double(p->tau), cs));
    launches += 3;
  }
  g_launches = launches;
  return ADAHOP_OK;
}

adahop_status_t adahop_calibrate_batch_outliers(int32_t n, const int64_t* rows, const int64_t* cols, const void* ws,
                                                size_t ws_bytes, double kappa, int32_t* d_counts,
                                                adahop_stream_t stream) {
  if (n <= 0 || !rows || !cols || !ws || !d_counts || !(kappa > 0)) return ADAHOP_E_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (rows[i] <= 0 || cols[i] <= 0) return ADAHOP_E_SHAPE;
  if (ws_bytes < adahop_calibrate_batch_workspace_bytes(n, rows, cols) || (reinterpret_cast<uintptr_t>(ws) & 255))
    return ADAHOP_E_WORKSPACE;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  const uint8_t* base = static_cast<const uint8_t*>(ws);
  int32_t launches = 0;
  for (int32_t i0 = 0; i0 < n; i0 += kCalibMaxJobs) {
    CalibJob jobs[kCalibMaxJobs];
    const int m = int(std::min<int32_t>(kCalibMaxJobs, n - i0));
    for (int k = 0; k < m; ++k) {
      const int32_t i = i0 + k;
      Carver c;   // rs and cs of adahop_calibrate's layout
      double* rs = reinterpret_cast<double*>(const_cast<uint8_t*>(base) + c.take(size_t(rows[i]) * 32));
      double* csum = reinterpret_cast<double*>(const_cast<uint8_t*>(base) + c.take(size_t(cols[i]) * 32));
      jobs[k] = CalibJob{nullptr, rows[i], cols[i], cols[i], rs, csum, nullptr, nullptr, nullptr, nullptr};
      base += (adahop_calibrate_workspace_bytes(rows[i], cols[i]) + 255) & ~size_t(255);
    }
    ADAHOP_LAUNCH(launch_outlier_counts_batch(jobs, m, kappa, d_counts + 2 * int64_t(i0),
                                              reinterpret_cast<cudaStream_t>(stream)));
    ++launches;
  }
  g_launches = launches;
  return ADAHOP_OK;
}

// ------------------------------------------------------------------------ hot path
size_t adahop_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, adahop_strategy_t s,
                                   const adahop_params_t* p) {
  if (!p || M <= 0 || N <= 0 || K <= 0) return 0;
  DevInfo d = dev_info();
  GemmPlan g;
  plan_gemm(M, N, K, s, p, d.ok ? d.sms : 148, &g);
  return g.total;
}

adahop_status_t adahop_gemm(const void* A, int32_t a_kstrided, int64_t lda, const void* B,
                            int32_t b_kstrided, int64_t ldb, void* C, adahop_dtype_t out_dt,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, adahop_strategy_t s,
                            const adahop_params_t* p, void* ws, size_t ws_bytes,
                            adahop_stream_t stream) {
  // ---- host-side validation (no launch happens before all checks pass)
  if (!A || !B || !C || !p) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = validate_params(p);
  if (st != ADAHOP_OK) return st;
  if (s < ADAHOP_IHT || s > ADAHOP_BF16) return ADAHOP_E_INVALID_ARG;
  if (out_dt != ADAHOP_DT_BF16 && out_dt != ADAHOP_DT_F32) return ADAHOP_E_INVALID_ARG;
  if (M <= 0 || N <= 0 || K <= 0) return ADAHOP_E_SHAPE;
  if (K % 32 != 0) return ADAHOP_E_SHAPE;
  if (M * (K / 64 + 1) >= (int64_t(1) << 31) || N * (K / 64 + 1) >= (int64_t(1) << 31))
    return ADAHOP_E_UNSUPPORTED;   // 32-bit block indexing in the quant kernels
  if ((a_kstrided != 0 && a_kstrided != 1) || (b_kstrided != 0 && b_kstrided != 1))
    return ADAHOP_E_INVALID_ARG;
  if (lda < (a_kstrided ? M : K) || ldb < (b_kstrided ? N : K) || ldc < N) return ADAHOP_E_INVALID_ARG;
  if ((lda % 8) || (ldb % 8) || !aligned16(A) || !aligned16(B) || !aligned16(C))
    return ADAHOP_E_INVALID_ARG;
  DevInfo dev;
  st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  GemmPlan g;
  plan_gemm(M, N, K, s, p, dev.sms, &g);
  if (!ws || ws_bytes < g.total || (reinterpret_cast<uintptr_t>(ws) & 255)) return ADAHOP_E_WORKSPACE;
  if (g.kk > 0 && g.rows_oe > kFoidMaxRows) return ADAHOP_E_UNSUPPORTED;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  const bool out_f32 = out_dt == ADAHOP_DT_F32;
  int32_t launches = 0;

  stage_mark(0, cs);
  // ---- Lv2 CC: the whole product in BF16
  if (s == ADAHOP_BF16) {
    Bf16GemmArgs ga{};
    ga.A = static_cast<const __nv_bfloat16*>(A); ga.a_mn = a_kstrided; ga.lda = lda;
    ga.B = static_cast<const __nv_bfloat16*>(B); ga.b_mn = b_kstrided; ga.ldb = ldb;
    ga.Mb = M; ga.Nb = N; ga.K = K; ga.mode = 0; ga.C = C; ga.out_f32 = out_f32; ga.ldc = ldc;
    stage_mark(1, cs);
    stage_mark(2, cs);
    ADAHOP_LAUNCH(run_gemm_bf16_full(ga, dev.sms, cs));
    stage_mark(3, cs);
    stage_mark(4, cs);
    g_launches = 1;
    return ADAHOP_OK;
  }

  uint8_t* qa = w + g.qa_codes;
  uint8_t* qa_sf = w + g.qa_sf;
  uint8_t* qb = w + g.qb_codes;
  uint8_t* qb_sf = w + g.qb_sf;
  int32_t* idx = g.kk > 0 ? reinterpret_cast<int32_t*>(w + g.idx) : nullptr;
  const bool oe_left = g.kk > 0 && s == ADAHOP_OE_LEFT_IHT;
  const bool oe_right = g.kk > 0 && s == ADAHOP_OE_RIGHT_IHT;

  // Scale-factor padding (rows beyond R or K beyond the last 256-block) must hold finite
  // scales: the padded codes are zero-filled by TMA, zero x finite scale = 0.
  if ((M % 128) || (K % 256)) ADAHOP_LAUNCH(cudaMemsetAsync(qa_sf, 0, size_t(sf_bytes(M, K)), cs));
  if ((N % 128) || (K % 256)) ADAHOP_LAUNCH(cudaMemsetAsync(qb_sf, 0, size_t(sf_bytes(N, K)), cs));

  // ---- 1. FOID (P:760 stage 1): probe keys + top-k indices (device-resident)
  const void* oe_src = oe_left ? A : B;
  const int oe_ks = oe_left ? a_kstrided : b_kstrided;
  const int64_t oe_ld = oe_left ? lda : ldb;
  __nv_bfloat16* slice = g.kk > 0 ? reinterpret_cast<__nv_bfloat16*>(w + g.slice) : nullptr;
  if (g.kk > 0) {
    ADAHOP_LAUNCH(launch_foid(oe_src, false, g.rows_oe, K, oe_ld, oe_ks, g.kk, p->foid_probe,
                              reinterpret_cast<double*>(w + g.keys), idx, cs));
    launches += foid_launches(g.rows_oe, K, p->foid_probe);
  }
  stage_mark(1, cs);
  // ---- 2. IHT + MXFP4 quantisation of both operands (P:761 stage 2); the OE rows are
  //         zeroed in the residual and gathered into the BF16 outlier slice in the same pass
  ADAHOP_LAUNCH(launch_iht_quant(A, false, M, K, lda, a_kstrided, oe_left ? idx : nullptr,
                                 oe_left ? g.kk : 0, qa, qa_sf, nullptr, oe_left ? slice : nullptr,
                                 false, dev.sms, cs));
  launches += quant_last_launches();
  ADAHOP_LAUNCH(launch_iht_quant(B, false, N, K, ldb, b_kstrided, oe_right ? idx : nullptr,
                                 oe_right ? g.kk : 0, qb, qb_sf, nullptr, oe_right ? slice : nullptr,
                                 false, dev.sms, cs));
  launches += quant_last_launches();
  stage_mark(2, cs);
  // ---- 3. BF16 outlier GEMM: split-K partials, written into C by the GEMM epilogue
  OePatch patch{};
  if (g.kk > 0) {
    Bf16GemmArgs ga{};
    if (oe_right) {  // D[M x k] = A (M x K) . B_out^T
      ga.A = static_cast<const __nv_bfloat16*>(A); ga.a_mn = a_kstrided; ga.lda = lda;
    } else {         // D[N x k] = B_store (N x K) . A_out^T  (transposed OE-Left product)
      ga.A = static_cast<const __nv_bfloat16*>(B); ga.a_mn = b_kstrided; ga.lda = ldb;
    }
    ga.B = slice; ga.b_mn = 0; ga.ldb = K;
    ga.Mb = g.mbig; ga.Nb = g.kk; ga.K = K; ga.mode = 1;
    ga.part = reinterpret_cast<float*>(w + g.part); ga.splits = g.splits; ga.npad = g.npad;
    float* Dt = reinterpret_cast<float*>(w + g.dt);
    ga.Dt = Dt;   // one K range: the GEMM writes Dt itself
    ADAHOP_LAUNCH(launch_gemm_bf16(ga, cs));
    launches += 1;
    if (ga.splits > 1) {
      ADAHOP_LAUNCH(launch_outlier_fold(ga.part, ga.splits, ga.Mb, ga.npad, g.kk, Dt, cs));
      launches += 1;
    }
    patch = OePatch{Dt, idx, ga.Mb, g.kk, oe_right ? 1 : 2};
  }
  stage_mark(3, cs);
  // ---- 4. block-scaled MXFP4 GEMM (P:762 stage 3); its epilogue writes the outlier entries
  //         (fused scatter: the residual product is exactly zero there)
  Mxf4GemmArgs ma{qa, qa_sf, qb, qb_sf, C, out_f32, ldc, M, N, K, patch};
  ADAHOP_LAUNCH(run_gemm_mxf4(ma, dev.sms, cs));
  launches += 1;
  stage_mark(4, cs);
  g_launches = launches;
  return ADAHOP_OK;
}

// ------------------------------------------------------------------------ layer step
// One linear layer's three matmuls with each operand tensor read ONCE by the
// dual-orientation quantiser (X: fwd + wgrad, W: fwd + dgrad, G_Y: dgrad + wgrad), either in one
// call (adahop_linear_layer) or split into the forward and the backward of a training step
// (adahop_linear_forward / adahop_linear_backward) with a caller-owned context in between.
}  // extern "C"

namespace {

// A carved buffer: byte offset in the workspace (space 0) or in the saved context (space 1).
struct Buf {
  size_t off = 0;
  int space = 0;
};

struct LayerPlan {
  // per tensor (0 = X [T x d_in], 1 = W [d_out x d_in], 2 = G_Y [T x d_out])
  int64_t R[3], C[3];
  bool need_row[3], need_col[3];
  Buf q_row[3], sf_row[3], q_col[3], sf_col[3];
  // masks: which FOID feeds which (tensor, orientation)
  int kk_row[3], kk_col[3];
  Buf idx_row[3], idx_col[3], slice_row[3], slice_col[3];
  Buf keys_row[3], keys_col[3];   // per-FOID scratch
  Buf part[3], dt[3];             // per-path outlier split-K partials and folded Dt
  int or_kk = 0;                  // the wgrad's outlier product fused into a quant pass (0: not planned)
  int or_t = -1;                  // the streamed tensor: G_Y (OE-Right) or X (OE-Left, layer call only)
  Buf or_part, or_ticket;         // its per-(band, CTA) partials; the GEMM pre-fold's CTA count
  int od_kk = 0;                  // the dgrad's OE-Left product fused into W's quant pass (layer call)
  Buf od_part, od_ticket;
  int splits[3];
  int64_t npad[3], mbig[3];
  size_t ws_total = 0, ctx_total = 0;
};

struct Spaces {
  uint8_t* base[2];
  template <typename T>
  T* p(const Buf& b) const { return reinterpret_cast<T*>(base[b.space] + b.off); }
};

// path p: (A tensor, A orientation, B tensor, B orientation); orientation 0 = row, 1 = col
constexpr int kPathA[3] = {0, 2, 2}, kPathAo[3] = {0, 0, 1};
constexpr int kPathB[3] = {1, 1, 0}, kPathBo[3] = {0, 1, 1};
// phases: the forward prepares X and W and runs path 0; the backward prepares G_Y and runs 1, 2
constexpr int kFwd = 1, kBwd = 2;
inline int tensor_phase(int t) { return t == 2 ? kBwd : kFwd; }
inline int path_phase(int path) { return path == 0 ? kFwd : kBwd; }

// split: the buffers the forward produces for the backward — the column (K = tokens / d_out)
// FP4 layouts of X and W with their OE indices and BF16 slices — are carved in the context.
void plan_layer(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s, const adahop_params_t* p,
                int sms, bool split, LayerPlan* L) {
  *L = LayerPlan{};
  L->R[0] = T; L->C[0] = d_in;
  L->R[1] = d_out; L->C[1] = d_in;
  L->R[2] = T; L->C[2] = d_out;
  for (int t = 0; t < 3; ++t) { L->kk_row[t] = L->kk_col[t] = 0; L->need_row[t] = L->need_col[t] = false; }
  for (int path = 0; path < 3; ++path) {
    if (s[path] == ADAHOP_BF16) continue;
    const int ta = kPathA[path], tb = kPathB[path];
    (kPathAo[path] ? L->need_col : L->need_row)[ta] = true;
    (kPathBo[path] ? L->need_col : L->need_row)[tb] = true;
    if (p->oe_k > 0 && (s[path] == ADAHOP_OE_LEFT_IHT || s[path] == ADAHOP_OE_RIGHT_IHT)) {
      const bool left = s[path] == ADAHOP_OE_LEFT_IHT;
      const int t = left ? ta : tb;
      const int o = left ? kPathAo[path] : kPathBo[path];
      const int64_t rows = o ? L->C[t] : L->R[t];        // stored rows of the OE operand
      const int kk = int(std::min<int64_t>(p->oe_k, rows));
      (o ? L->kk_col : L->kk_row)[t] = kk;
    }
  }
  Carver c[2];
  auto take = [&](Buf& b, size_t bytes, bool ctx) {
    b.space = ctx ? 1 : 0;
    b.off = c[b.space].take(bytes);
  };
  for (int t = 0; t < 3; ++t) {
    const int64_t R = L->R[t], C = L->C[t];
    const bool keep = split && t != 2;   // X / W column layouts outlive the forward
    if (L->need_row[t]) { take(L->q_row[t], size_t(R) * size_t(C / 2), false); take(L->sf_row[t], size_t(sf_bytes(R, C)), false); }
    if (L->need_col[t]) { take(L->q_col[t], size_t(C) * size_t(R / 2), keep); take(L->sf_col[t], size_t(sf_bytes(C, R)), keep); }
    if (L->kk_row[t]) {
      take(L->idx_row[t], size_t(L->kk_row[t]) * 4, false);
      take(L->slice_row[t], size_t(L->kk_row[t]) * size_t(C) * 2, false);
      take(L->keys_row[t], foid_ws_bytes(R), false);
    }
    if (L->kk_col[t]) {
      take(L->idx_col[t], size_t(L->kk_col[t]) * 4, keep);
      take(L->slice_col[t], size_t(L->kk_col[t]) * size_t(R) * 2, keep);
      take(L->keys_col[t], foid_ws_bytes(C), false);
    }
  }
  const int64_t MNK[3][3] = {{T, d_out, d_in}, {T, d_in, d_out}, {d_out, d_in, T}};
  for (int path = 0; path < 3; ++path) {
    L->splits[path] = 1; L->npad[path] = 0; L->mbig[path] = 0;
    if (p->oe_k <= 0 || (s[path] != ADAHOP_OE_LEFT_IHT && s[path] != ADAHOP_OE_RIGHT_IHT)) continue;
    const bool left = s[path] == ADAHOP_OE_LEFT_IHT;
    const int t = left ? kPathA[path] : kPathB[path];
    const int kk = (left ? kPathAo[path] : kPathBo[path]) ? L->kk_col[t] : L->kk_row[t];
    L->mbig[path] = left ? MNK[path][1] : MNK[path][0];
    L->npad[path] = bf16_gemm_npad(kk);
    L->splits[path] = bf16_gemm_splits(L->mbig[path], MNK[path][2], sms);
    take(L->part[path], size_t(L->splits[path]) * size_t(L->mbig[path]) * size_t(L->npad[path]) * 4, false);
    take(L->dt[path], size_t(kk) * size_t(L->mbig[path]) * 4, false);
  }
  // The wgrad's outlier product accumulates in a quant pass that streams its big operand anyway
  // ("fuses ... into a single kernel"), when that tensor is quantised in both orientations:
  //   OE-Right (A = G_Y^T, B_out = X[:, S]): G_Y's pass, slice = X's columns S;
  //   OE-Left (A_out = G_Y[:, S]^T, B = X): X's pass, slice = G_Y's columns S — only when X and G_Y
  //   share the launch (the layer call; the split backward has no X pass and uses the BF16 GEMM).
  const bool right = s[2] == ADAHOP_OE_RIGHT_IHT, left = s[2] == ADAHOP_OE_LEFT_IHT;
  const int ot = right ? 2 : 0, st_ = right ? 0 : 2;   // streamed tensor, slice's tensor
  if (or_fusion_enabled() && (right || (left && !split && or_left_enabled())) && p->oe_k > 0 && L->kk_col[st_] > 0 &&
      L->need_row[ot] && L->need_col[ot]) {
    const size_t b = quant_tc_or_part_bytes(L->R[ot], L->C[ot], L->kk_col[st_], sms);
    if (b > 0) {
      L->or_kk = L->kk_col[st_];
      L->or_t = ot;
      take(L->or_part, b, false);
      take(L->or_ticket, 4, false);
    }
  }
  // The dgrad's OE-Left product (A_out = G_Y[S, :], B = W^T stored: C_out = G_Y[S, :] W, eq:oe_left
  // P:273) streams W, which the layer call quantises in both orientations: W's pass accumulates it
  // with G_Y's row slice (gathered before the launch) as the product's second operand
  if (or_fusion_enabled() && or_dgrad_enabled() && !split && s[1] == ADAHOP_OE_LEFT_IHT && p->oe_k > 0 &&
      L->kk_row[2] > 0 && L->need_row[1] && L->need_col[1]) {
    const size_t b = quant_tc_or_part_bytes(L->R[1], L->C[1], L->kk_row[2], sms);
    if (b > 0) {
      L->od_kk = L->kk_row[2];
      take(L->od_part, b, false);
      take(L->od_ticket, 4, false);
    }
  }
  L->ws_total = c[0].take(0) + 256;
  L->ctx_total = split ? c[1].take(0) + 256 : 0;
}

// The backward reads the full X in BF16 only for a wgrad whose BF16 part multiplies by all of X:
// OE-Left (A_out . B with B = X) and the Lv2 BF16 wgrad. Everything else the
// backward needs from the forward is in the context (FP4 + BF16 outlier slices).
bool backward_needs_x(const adahop_strategy_t* s, const adahop_params_t* p) {
  return s[2] == ADAHOP_BF16 || (s[2] == ADAHOP_OE_LEFT_IHT && p->oe_k > 0);
}

adahop_status_t check_layer_args(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                 const adahop_params_t* p, std::initializer_list<const void*> ptrs) {
  if (!s || !p) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = validate_params(p);
  if (st != ADAHOP_OK) return st;
  for (int i = 0; i < 3; ++i)
    if (s[i] < ADAHOP_IHT || s[i] > ADAHOP_BF16) return ADAHOP_E_INVALID_ARG;
  if (T <= 0 || d_in <= 0 || d_out <= 0) return ADAHOP_E_SHAPE;
  if (T % 32 || d_in % 32 || d_out % 32) return ADAHOP_E_SHAPE;
  for (const void* q : ptrs)
    if (!q || !aligned16(q)) return ADAHOP_E_INVALID_ARG;
  if (T * (std::max(d_in, d_out) / 64 + 1) >= (int64_t(1) << 31)) return ADAHOP_E_UNSUPPORTED;
  return ADAHOP_OK;
}

adahop_status_t check_oe_rows(const LayerPlan& L, int phases) {
  for (int t = 0; t < 3; ++t) {
    if (!(tensor_phase(t) & phases)) continue;
    if (L.kk_row[t] && L.R[t] > kFoidMaxRows) return ADAHOP_E_UNSUPPORTED;
    if (L.kk_col[t] && L.C[t] > kFoidMaxRows) return ADAHOP_E_UNSUPPORTED;
  }
  return ADAHOP_OK;
}

// The layer's kernels for the given phases. Inputs a phase does not use may be NULL; out[path]
// is written in odt[path].
adahop_status_t run_layer(int phases, const void* X, const void* W, const void* GY, void* const out[3],
                          const adahop_dtype_t odt[3], int64_t T, int64_t d_in, int64_t d_out,
                          const adahop_strategy_t* s, const adahop_params_t* p, const LayerPlan& L,
                          const Spaces& sp, int sms, cudaStream_t cs) {
  const __nv_bfloat16* src[3] = {static_cast<const __nv_bfloat16*>(X), static_cast<const __nv_bfloat16*>(W),
                                 static_cast<const __nv_bfloat16*>(GY)};
  int32_t launches = 0;
  stage_mark(0, cs);
  // ---- 1. FOID for every OE operand of these phases: row orientation = rows of the
  //         tensor (K-contiguous probe), column orientation = columns (probe = first 64 rows)
  {
    FoidJob jobs[kFoidMaxJobs];
    int nj = 0;
    for (int t = 0; t < 3; ++t) {
      if (!(tensor_phase(t) & phases)) continue;
      if (L.kk_row[t])
        jobs[nj++] = FoidJob{src[t], L.R[t], L.C[t], L.C[t], 0, L.kk_row[t], p->foid_probe,
                             sp.p<double>(L.keys_row[t]), sp.p<int32_t>(L.idx_row[t])};
      if (L.kk_col[t])
        jobs[nj++] = FoidJob{src[t], L.C[t], L.R[t], L.C[t], 1, L.kk_col[t], p->foid_probe,
                             sp.p<double>(L.keys_col[t]), sp.p<int32_t>(L.idx_col[t])};
    }
    if (nj) {
      ADAHOP_LAUNCH(launch_foid_batch(jobs, nj, false, cs));
      launches += 2;
    }
  }
  stage_mark(1, cs);
  // ---- 2. one quantisation pass per tensor (both orientations when both are consumed); the
  //         tensors that need both orientations share ONE persistent tensor-core launch
  QuantTcJob tc_jobs[3];
  int tc_t[3];   // tensor of each tc job
  int n_tc = 0;
  bool in_tc[3] = {false, false, false};
  // tensors quantised by the tensor-core pass: their OE slices are gathered before it (a fused
  // product may only take its slice from such a tensor, or from the saved context)
  bool will_tc[3];
  for (int t = 0; t < 3; ++t)
    will_tc[t] = (tensor_phase(t) & phases) && L.need_row[t] && L.need_col[t] && quant_use_tc() &&
                 quant_tc_supported(L.R[t], L.C[t], L.C[t], src[t], L.kk_row[t] > 0, L.kk_col[t] > 0);
  for (int t = 0; t < 3; ++t) {
    if (!will_tc[t]) continue;
    const int64_t R = L.R[t], C = L.C[t];
    in_tc[t] = true;
    tc_t[n_tc] = t;
    tc_jobs[n_tc++] = QuantTcJob{
        src[t], R, C, C,
        L.kk_row[t] ? sp.p<const int32_t>(L.idx_row[t]) : nullptr, L.kk_row[t],
        L.kk_row[t] ? sp.p<__nv_bfloat16>(L.slice_row[t]) : nullptr, sp.p<uint8_t>(L.q_row[t]), sp.p<uint8_t>(L.sf_row[t]),
        nullptr,
        L.kk_col[t] ? sp.p<const int32_t>(L.idx_col[t]) : nullptr, L.kk_col[t],
        L.kk_col[t] ? sp.p<__nv_bfloat16>(L.slice_col[t]) : nullptr, sp.p<uint8_t>(L.q_col[t]), sp.p<uint8_t>(L.sf_col[t]),
        nullptr};
    // OE-Right's slice (X's columns) is in this call or the saved context; OE-Left's (G_Y's columns)
    // is gathered before this launch when G_Y is in it
    if (t == L.or_t && L.or_kk > 0 && (t == 2 ? !(phases & tensor_phase(0)) || will_tc[0] : will_tc[2])) {
      QuantTcJob& q = tc_jobs[n_tc - 1];
      q.or_slice = sp.p<const __nv_bfloat16>(L.slice_col[2 - t]);
      q.or_kk = L.or_kk;
      q.or_part = sp.p<float>(L.or_part);
      q.or_part_bytes = quant_tc_or_part_bytes(R, C, L.or_kk, sms);
      q.or_ticket = sp.p<unsigned>(L.or_ticket);
    }
    // the dgrad's OE-Left product in W's pass (G_Y's row slice is gathered before this launch)
    if (t == 1 && L.od_kk > 0 && will_tc[2]) {
      QuantTcJob& q = tc_jobs[n_tc - 1];
      q.or_slice = sp.p<const __nv_bfloat16>(L.slice_row[2]);
      q.or_kk = L.od_kk;
      q.or_part = sp.p<float>(L.od_part);
      q.or_part_bytes = quant_tc_or_part_bytes(R, C, L.od_kk, sms);
      q.or_ticket = sp.p<unsigned>(L.od_ticket);
    }
    if ((R % 128) || (C % 256)) ADAHOP_LAUNCH(cudaMemsetAsync(sp.p<uint8_t>(L.sf_row[t]), 0, size_t(sf_bytes(R, C)), cs));
    if ((C % 128) || (R % 256)) ADAHOP_LAUNCH(cudaMemsetAsync(sp.p<uint8_t>(L.sf_col[t]), 0, size_t(sf_bytes(C, R)), cs));
  }
  bool fused_t[3] = {false, false, false};   // the tensor's pass carried its fused product
  if (n_tc) {
    int nl = 0;
    bool fj[3] = {false, false, false};
    ADAHOP_LAUNCH(launch_quant_tc_multi(tc_jobs, n_tc, sms, cs, &nl, fj));
    for (int i = 0; i < n_tc; ++i) fused_t[tc_t[i]] = fj[i];
    launches += nl;
  }
  const bool or_fused = L.or_kk > 0 && L.or_t >= 0 && fused_t[L.or_t];
  const bool od_fused = L.od_kk > 0 && fused_t[1];
  for (int t = 0; t < 3; ++t) {
    if (!(tensor_phase(t) & phases) || in_tc[t]) continue;
    const int64_t R = L.R[t], C = L.C[t];
    const int32_t* rz = L.kk_row[t] ? sp.p<const int32_t>(L.idx_row[t]) : nullptr;
    const int32_t* cz = L.kk_col[t] ? sp.p<const int32_t>(L.idx_col[t]) : nullptr;
    __nv_bfloat16* srow = L.kk_row[t] ? sp.p<__nv_bfloat16>(L.slice_row[t]) : nullptr;
    __nv_bfloat16* scol = L.kk_col[t] ? sp.p<__nv_bfloat16>(L.slice_col[t]) : nullptr;
    uint8_t *qr = sp.p<uint8_t>(L.q_row[t]), *sr = sp.p<uint8_t>(L.sf_row[t]);
    uint8_t *qc = sp.p<uint8_t>(L.q_col[t]), *sc = sp.p<uint8_t>(L.sf_col[t]);
    if (L.need_row[t] && ((R % 128) || (C % 256))) ADAHOP_LAUNCH(cudaMemsetAsync(sr, 0, size_t(sf_bytes(R, C)), cs));
    if (L.need_col[t] && ((C % 128) || (R % 256))) ADAHOP_LAUNCH(cudaMemsetAsync(sc, 0, size_t(sf_bytes(C, R)), cs));
    if (L.need_row[t] && L.need_col[t] && dual_quant_supported(R, C, rz != nullptr, cz != nullptr)) {
      ADAHOP_LAUNCH(launch_iht_quant_dual(src[t], R, C, C, rz, L.kk_row[t], srow, qr, sr, cz, L.kk_col[t], scol, qc, sc,
                                          sms, cs));
      launches += quant_last_launches();
    } else {
      if (L.need_row[t]) {
        ADAHOP_LAUNCH(launch_iht_quant(src[t], false, R, C, C, 0, rz, L.kk_row[t], qr, sr, nullptr, srow, false, sms, cs));
        launches += quant_last_launches();
      }
      if (L.need_col[t]) {
        ADAHOP_LAUNCH(launch_iht_quant(src[t], false, C, R, C, 1, cz, L.kk_col[t], qc, sc, nullptr, scol, false, sms, cs));
        launches += quant_last_launches();
      }
    }
  }
  stage_mark(2, cs);
  const int64_t MNK[3][3] = {{T, d_out, d_in}, {T, d_in, d_out}, {d_out, d_in, T}};
  const int64_t ldc[3] = {d_out, d_in, d_in};
  // raw operand views per path: A_store / B_store as (ptr, kstrided, ld)
  const void* rawA[3] = {X, GY, GY};
  const int rawAks[3] = {0, 0, 1};
  const int64_t rawAld[3] = {d_in, d_out, d_out};
  const void* rawB[3] = {W, W, X};
  const int rawBks[3] = {0, 1, 1};
  const int64_t rawBld[3] = {d_in, d_in, d_in};
  // ---- 3. BF16 outlier GEMMs: split-K partials, written into C by the MXFP4 GEMM epilogue
  OePatch patch[3] = {};
  for (int path = 0; path < 3; ++path) {
    if (!(path_phase(path) & phases) || L.mbig[path] == 0) continue;
    const bool left = s[path] == ADAHOP_OE_LEFT_IHT;
    const int t = left ? kPathA[path] : kPathB[path];
    const bool col = left ? kPathAo[path] : kPathBo[path];
    const int kk = col ? L.kk_col[t] : L.kk_row[t];
    const int32_t* idx = sp.p<const int32_t>(col ? L.idx_col[t] : L.idx_row[t]);
    if (path == 2 && or_fused) {   // the quant pass left the product's partials; the epilogue sums them
      patch[path] = quant_tc_or_patch(L.R[L.or_t], L.C[L.or_t], kk, sms, sp.p<const float>(L.or_part),
                                      sp.p<unsigned>(L.or_ticket), sp.p<float>(L.dt[path]), idx, left ? 2 : 1);
      continue;
    }
    if (path == 1 && od_fused) {   // the dgrad's OE-Left product from W's pass (rows idx of G_X)
      patch[path] = quant_tc_or_patch(L.R[1], L.C[1], kk, sms, sp.p<const float>(L.od_part),
                                      sp.p<unsigned>(L.od_ticket), sp.p<float>(L.dt[path]), idx, 2);
      continue;
    }
    const __nv_bfloat16* slice = sp.p<const __nv_bfloat16>(col ? L.slice_col[t] : L.slice_row[t]);
    Bf16GemmArgs ga{};
    if (!left) { ga.A = static_cast<const __nv_bfloat16*>(rawA[path]); ga.a_mn = rawAks[path]; ga.lda = rawAld[path]; }
    else { ga.A = static_cast<const __nv_bfloat16*>(rawB[path]); ga.a_mn = rawBks[path]; ga.lda = rawBld[path]; }
    ga.B = slice; ga.b_mn = 0; ga.ldb = MNK[path][2];
    ga.Mb = L.mbig[path]; ga.Nb = kk; ga.K = MNK[path][2]; ga.mode = 1;
    ga.part = sp.p<float>(L.part[path]); ga.splits = L.splits[path]; ga.npad = L.npad[path];
    float* Dt = sp.p<float>(L.dt[path]);
    ga.Dt = Dt;   // one K range: the GEMM writes Dt itself
    ADAHOP_LAUNCH(launch_gemm_bf16(ga, cs));
    launches += 1;
    if (ga.splits > 1) {
      ADAHOP_LAUNCH(launch_outlier_fold(ga.part, ga.splits, ga.Mb, ga.npad, kk, Dt, cs));
      launches += 1;
    }
    patch[path] = OePatch{Dt, idx, ga.Mb, kk, left ? 2 : 1};
  }
  stage_mark(3, cs);
  // ---- 4. the MXFP4 GEMMs (or BF16 for Lv2 CC); the epilogue writes the outlier entries
  Mxf4GemmArgs group[3];
  int ng = 0;
  for (int path = 0; path < 3; ++path) {
    if (!(path_phase(path) & phases)) continue;
    const int64_t M = MNK[path][0], N = MNK[path][1], K = MNK[path][2];
    const bool f32 = odt[path] == ADAHOP_DT_F32;
    if (s[path] == ADAHOP_BF16) {
      Bf16GemmArgs ga{};
      ga.A = static_cast<const __nv_bfloat16*>(rawA[path]); ga.a_mn = rawAks[path]; ga.lda = rawAld[path];
      ga.B = static_cast<const __nv_bfloat16*>(rawB[path]); ga.b_mn = rawBks[path]; ga.ldb = rawBld[path];
      ga.Mb = M; ga.Nb = N; ga.K = K; ga.mode = 0; ga.C = out[path]; ga.out_f32 = f32; ga.ldc = ldc[path];
      ADAHOP_LAUNCH(run_gemm_bf16_full(ga, sms, cs));
      launches += 1;
      continue;
    }
    const int ta = kPathA[path], tb = kPathB[path];
    const uint8_t* qa = sp.p<const uint8_t>(kPathAo[path] ? L.q_col[ta] : L.q_row[ta]);
    const uint8_t* qa_sf = sp.p<const uint8_t>(kPathAo[path] ? L.sf_col[ta] : L.sf_row[ta]);
    const uint8_t* qb = sp.p<const uint8_t>(kPathBo[path] ? L.q_col[tb] : L.q_row[tb]);
    const uint8_t* qb_sf = sp.p<const uint8_t>(kPathBo[path] ? L.sf_col[tb] : L.sf_row[tb]);
    Mxf4GemmArgs ma{qa, qa_sf, qb, qb_sf, out[path], f32, ldc[path], M, N, K, patch[path]};
    group[ng++] = ma;
  }
  // A small linear's GEMMs share one persistent launch (clusters split by work); large ones, and
  // any with M <= 128 (the 1-CTA kernel), keep their own launches
  double flops = 0;
  bool pairs_ok = true;
  for (int i = 0; i < ng; ++i) {
    flops += 2.0 * double(group[i].M) * double(group[i].N) * double(group[i].K);
    pairs_ok &= group[i].M > 128;
  }
  bool grouped = false;
  if (ng >= 2 && pairs_ok && group_gemms(flops)) {
    ADAHOP_LAUNCH(launch_gemm_mxf4_2sm_group(group, ng, sms, cs, &grouped));
    if (grouped) launches += 1;
  }
  if (!grouped) {
    for (int i = 0; i < ng; ++i) {
      ADAHOP_LAUNCH(run_gemm_mxf4(group[i], sms, cs, false));
      launches += 1;
    }
  }
  stage_mark(4, cs);
  g_launches = launches;
  return ADAHOP_OK;
}

inline bool valid_dt(adahop_dtype_t d) { return d == ADAHOP_DT_BF16 || d == ADAHOP_DT_F32; }

}  // namespace

extern "C" {

size_t adahop_layer_workspace_bytes(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                    const adahop_params_t* p) {
  if (!s || !p || T <= 0 || d_in <= 0 || d_out <= 0) return 0;
  DevInfo d = dev_info();
  LayerPlan L;
  plan_layer(T, d_in, d_out, s, p, d.ok ? d.sms : 148, false, &L);
  return L.ws_total;
}

adahop_status_t adahop_linear_layer(const void* X, const void* W, const void* GY, void* Y, void* GX, void* GW,
                                    adahop_dtype_t out_dt, adahop_dtype_t gw_dt, int64_t T, int64_t d_in,
                                    int64_t d_out, const adahop_strategy_t* s, const adahop_params_t* p, void* ws,
                                    size_t ws_bytes, adahop_stream_t stream) {
  if (!valid_dt(out_dt) || !valid_dt(gw_dt)) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = check_layer_args(T, d_in, d_out, s, p, {X, W, GY, Y, GX, GW});
  if (st != ADAHOP_OK) return st;
  DevInfo dev;
  st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  LayerPlan L;
  plan_layer(T, d_in, d_out, s, p, dev.sms, false, &L);
  if (!ws || ws_bytes < L.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255)) return ADAHOP_E_WORKSPACE;
  st = check_oe_rows(L, kFwd | kBwd);
  if (st != ADAHOP_OK) return st;
  void* const out[3] = {Y, GX, GW};
  const adahop_dtype_t odt[3] = {out_dt, out_dt, gw_dt};
  const Spaces sp{{static_cast<uint8_t*>(ws), nullptr}};
  return run_layer(kFwd | kBwd, X, W, GY, out, odt, T, d_in, d_out, s, p, L, sp, dev.sms,
                   reinterpret_cast<cudaStream_t>(stream));
}

size_t adahop_linear_ctx_bytes(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                               const adahop_params_t* p) {
  if (!s || !p || T <= 0 || d_in <= 0 || d_out <= 0) return 0;
  DevInfo d = dev_info();
  LayerPlan L;
  plan_layer(T, d_in, d_out, s, p, d.ok ? d.sms : 148, true, &L);
  return L.ctx_total;
}

size_t adahop_linear_split_workspace_bytes(int64_t T, int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                           const adahop_params_t* p) {
  if (!s || !p || T <= 0 || d_in <= 0 || d_out <= 0) return 0;
  DevInfo d = dev_info();
  LayerPlan L;
  plan_layer(T, d_in, d_out, s, p, d.ok ? d.sms : 148, true, &L);
  return L.ws_total;
}

int32_t adahop_linear_backward_needs_x(const adahop_strategy_t* s, const adahop_params_t* p) {
  if (!s || !p) return 0;
  return backward_needs_x(s, p) ? 1 : 0;
}

adahop_status_t adahop_linear_forward(const void* X, const void* W, void* Y, adahop_dtype_t out_dt, int64_t T,
                                      int64_t d_in, int64_t d_out, const adahop_strategy_t* s,
                                      const adahop_params_t* p, void* ctx, size_t ctx_bytes, void* ws,
                                      size_t ws_bytes, adahop_stream_t stream) {
  if (!valid_dt(out_dt)) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = check_layer_args(T, d_in, d_out, s, p, {X, W, Y});
  if (st != ADAHOP_OK) return st;
  DevInfo dev;
  st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  LayerPlan L;
  plan_layer(T, d_in, d_out, s, p, dev.sms, true, &L);
  if (!ws || ws_bytes < L.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255)) return ADAHOP_E_WORKSPACE;
  if (!ctx || ctx_bytes < L.ctx_total || (reinterpret_cast<uintptr_t>(ctx) & 255)) return ADAHOP_E_WORKSPACE;
  st = check_oe_rows(L, kFwd);
  if (st != ADAHOP_OK) return st;
  void* const out[3] = {Y, nullptr, nullptr};
  const adahop_dtype_t odt[3] = {out_dt, out_dt, out_dt};
  const Spaces sp{{static_cast<uint8_t*>(ws), static_cast<uint8_t*>(ctx)}};
  return run_layer(kFwd, X, W, nullptr, out, odt, T, d_in, d_out, s, p, L, sp, dev.sms,
                   reinterpret_cast<cudaStream_t>(stream));
}

adahop_status_t adahop_linear_backward(const void* GY, const void* W, const void* X, void* GX, void* GW,
                                       adahop_dtype_t gx_dt, adahop_dtype_t gw_dt, int64_t T, int64_t d_in,
                                       int64_t d_out, const adahop_strategy_t* s, const adahop_params_t* p,
                                       const void* ctx, size_t ctx_bytes, void* ws, size_t ws_bytes,
                                       adahop_stream_t stream) {
  if (!valid_dt(gx_dt) || !valid_dt(gw_dt)) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = check_layer_args(T, d_in, d_out, s, p, {GY, W, GX, GW});
  if (st != ADAHOP_OK) return st;
  if (backward_needs_x(s, p) ? (!X || !aligned16(X)) : false) return ADAHOP_E_INVALID_ARG;
  DevInfo dev;
  st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  LayerPlan L;
  plan_layer(T, d_in, d_out, s, p, dev.sms, true, &L);
  if (!ws || ws_bytes < L.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255)) return ADAHOP_E_WORKSPACE;
  if (!ctx || ctx_bytes < L.ctx_total || (reinterpret_cast<uintptr_t>(ctx) & 255)) return ADAHOP_E_WORKSPACE;
  st = check_oe_rows(L, kBwd);
  if (st != ADAHOP_OK) return st;
  void* const out[3] = {nullptr, GX, GW};
  const adahop_dtype_t odt[3] = {gx_dt, gx_dt, gw_dt};
  const Spaces sp{{static_cast<uint8_t*>(ws), static_cast<uint8_t*>(const_cast<void*>(ctx))}};
  return run_layer(kBwd, backward_needs_x(s, p) ? X : nullptr, W, GY, out, odt, T, d_in, d_out, s, p, L, sp, dev.sms,
                   reinterpret_cast<cudaStream_t>(stream));
}

size_t adahop_workspace_bytes(adahop_path_t path, int64_t T, int64_t d_in, int64_t d_out,
                              adahop_strategy_t s, const adahop_params_t* p) {
  switch (path) {
    case ADAHOP_PATH_FWD: return adahop_gemm_workspace_bytes(T, d_out, d_in, s, p);
    case ADAHOP_PATH_DGRAD: return adahop_gemm_workspace_bytes(T, d_in, d_out, s, p);
    case ADAHOP_PATH_WGRAD: return adahop_gemm_workspace_bytes(d_out, d_in, T, s, p);
  }
  return 0;
}

adahop_status_t adahop_linear_fwd(const void* X, const void* W, void* Y, adahop_dtype_t out_dt,
                                  int64_t T, int64_t d_in, int64_t d_out, adahop_strategy_t s,
                                  const adahop_params_t* p, void* ws, size_t ws_bytes,
                                  adahop_stream_t stream) {
  // Y = X W^T: A_store = X (T x d_in), B_store = W (d_out x d_in)
  return adahop_gemm(X, 0, d_in, W, 0, d_in, Y, out_dt, d_out, T, d_out, d_in, s, p, ws, ws_bytes,
                     stream);
}

adahop_status_t adahop_linear_dgrad(const void* GY, const void* W, void* GX, adahop_dtype_t out_dt,
                                    int64_t T, int64_t d_in, int64_t d_out, adahop_strategy_t s,
                                    const adahop_params_t* p, void* ws, size_t ws_bytes,
                                    adahop_stream_t stream) {
  // G_X = G_Y W: A_store = G_Y (T x d_out), B_store = W^T (K-strided view of W)
  return adahop_gemm(GY, 0, d_out, W, 1, d_in, GX, out_dt, d_in, T, d_in, d_out, s, p, ws,
                     ws_bytes, stream);
}

adahop_status_t adahop_linear_wgrad(const void* GY, const void* X, void* GW, adahop_dtype_t out_dt,
                                    int64_t T, int64_t d_in, int64_t d_out, adahop_strategy_t s,
                                    const adahop_params_t* p, void* ws, size_t ws_bytes,
                                    adahop_stream_t stream) {
  // G_W = G_Y^T X: A_store = G_Y^T, B_store = X^T, both K-strided (K = tokens)
  if (T % 32 != 0) return ADAHOP_E_SHAPE;
  return adahop_gemm(GY, 1, d_out, X, 1, d_in, GW, out_dt, d_in, d_out, d_in, T, s, p, ws,
                     ws_bytes, stream);
}

// ------------------------------------------------------------------------ debug entry points
size_t adahop_debug_workspace_bytes(int64_t R, int64_t K) {
  if (R <= 0 || K <= 0) return 0;
  Carver c;
  c.take(size_t(sf_bytes(R, K)));
  c.take(foid_ws_bytes(R));                                // FOID keys + candidates
  return c.take(0) + 256;
}

adahop_status_t adahop_debug_iht_quant(const void* in, adahop_dtype_t dt, int64_t R, int64_t K,
                                       int64_t ld, int32_t k_strided, const int32_t* zero_rows,
                                       int32_t nzero, float* had_out, uint8_t* codes_canon,
                                       uint8_t* scales_canon, void* ws, size_t ws_bytes,
                                       adahop_stream_t stream) {
  if (!in || !codes_canon || !scales_canon || !ws) return ADAHOP_E_INVALID_ARG;
  if (nzero < 0 || (nzero > 0 && !zero_rows)) return ADAHOP_E_INVALID_ARG;
  if (R <= 0 || K <= 0 || K % 32) return ADAHOP_E_SHAPE;
  if (R * (K / 64 + 1) >= (int64_t(1) << 31)) return ADAHOP_E_UNSUPPORTED;
  const int64_t esz = dt == ADAHOP_DT_F32 ? 4 : 2;
  if (ld < (k_strided ? R : K)) return ADAHOP_E_INVALID_ARG;
  // the row kernel uses 16-byte vector loads; the transposing kernel checks alignment itself
  if (!k_strided && ((ld * esz) % 16 || !aligned16(in))) return ADAHOP_E_INVALID_ARG;
  if (ws_bytes < adahop_debug_workspace_bytes(R, K)) return ADAHOP_E_WORKSPACE;
  DevInfo dev;
  adahop_status_t st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* sf = static_cast<uint8_t*>(ws);
  ADAHOP_LAUNCH(launch_iht_quant(in, dt == ADAHOP_DT_F32, R, K, ld, k_strided, zero_rows, nzero,
                                 codes_canon, sf, had_out, nullptr, false, dev.sms, cs));
  ADAHOP_LAUNCH(launch_sf_convert(sf, R, K, scales_canon, true, cs));
  g_launches = 2;
  return ADAHOP_OK;
}

adahop_status_t adahop_debug_quant_dual(const void* in, adahop_dtype_t dt, int64_t R, int64_t C, int64_t ld,
                                       const int32_t* row_zero, int32_t nrow_zero, const int32_t* col_zero,
                                       int32_t ncol_zero, uint8_t* q_row, uint8_t* scales_row, uint8_t* q_col,
                                       uint8_t* scales_col, void* slice_row, void* slice_col, void* ws,
                                       size_t ws_bytes, adahop_stream_t stream) {
  if (!in || !q_row || !scales_row || !q_col || !scales_col || !ws) return ADAHOP_E_INVALID_ARG;
  if (dt != ADAHOP_DT_BF16) return ADAHOP_E_UNSUPPORTED;
  if (nrow_zero < 0 || ncol_zero < 0 || (nrow_zero > 0 && !row_zero) || (ncol_zero > 0 && !col_zero))
    return ADAHOP_E_INVALID_ARG;
  if (nrow_zero > 256 || ncol_zero > 256) return ADAHOP_E_UNSUPPORTED;
  if (R <= 0 || C <= 0 || R % 32 || C % 32) return ADAHOP_E_SHAPE;
  if (ld < C || (ld * 2) % 16 || !aligned16(in)) return ADAHOP_E_INVALID_ARG;
  if (ws_bytes < adahop_debug_workspace_bytes(R, C) + adahop_debug_workspace_bytes(C, R)) return ADAHOP_E_WORKSPACE;
  if (!dual_quant_supported(R, C, nrow_zero > 0, ncol_zero > 0)) return ADAHOP_E_UNSUPPORTED;
  DevInfo dev;
  adahop_status_t st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* sf_r = static_cast<uint8_t*>(ws);
  uint8_t* sf_c = sf_r + adahop_debug_workspace_bytes(R, C);
  ADAHOP_LAUNCH(launch_iht_quant_dual(static_cast<const __nv_bfloat16*>(in), R, C, ld, row_zero, nrow_zero,
                                      static_cast<__nv_bfloat16*>(slice_row), q_row, sf_r, col_zero, ncol_zero,
                                      static_cast<__nv_bfloat16*>(slice_col), q_col, sf_c, dev.sms, cs));
  ADAHOP_LAUNCH(launch_sf_convert(sf_r, R, C, scales_row, true, cs));
  ADAHOP_LAUNCH(launch_sf_convert(sf_c, C, R, scales_col, true, cs));
  g_launches = 3;
  return ADAHOP_OK;
}

adahop_status_t adahop_debug_foid(const void* in, adahop_dtype_t dt, int64_t R, int64_t K,
                                  int64_t ld, int32_t k_strided, int32_t k, int32_t probe,
                                  int32_t* idx_sorted, double* keys_out, void* ws, size_t ws_bytes,
                                  adahop_stream_t stream) {
  if (!in || !idx_sorted || !ws) return ADAHOP_E_INVALID_ARG;
  if (R <= 0 || K <= 0) return ADAHOP_E_SHAPE;
  if (k < 1 || k > 256 || probe < 1) return ADAHOP_E_UNSUPPORTED;
  if (ld < (k_strided ? R : K)) return ADAHOP_E_INVALID_ARG;
  if (ws_bytes < adahop_debug_workspace_bytes(R, K)) return ADAHOP_E_WORKSPACE;
  const int64_t kk = std::min<int64_t>(k, R);
  if (R > kFoidMaxRows) return ADAHOP_E_UNSUPPORTED;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  Carver c;
  uint8_t* w = static_cast<uint8_t*>(ws);
  c.take(size_t(sf_bytes(R, K)));
  double* keys = reinterpret_cast<double*>(w + c.take(foid_ws_bytes(R)));
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  ADAHOP_LAUNCH(launch_foid(in, dt == ADAHOP_DT_F32, R, K, ld, k_strided, int(kk), probe, keys,
                            idx_sorted, cs));
  if (keys_out)
    ADAHOP_LAUNCH(cudaMemcpyAsync(keys_out, keys, size_t(R) * 8, cudaMemcpyDeviceToDevice, cs));
  g_launches = 3;
  return ADAHOP_OK;
}

size_t adahop_debug_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  Carver c;
  c.take(size_t(sf_bytes(M, K)));
  c.take(size_t(sf_bytes(N, K)));
  return c.take(0) + 256;
}

adahop_status_t adahop_debug_gemm_mxf4(const uint8_t* a_codes, const uint8_t* a_scales,
                                       const uint8_t* b_codes, const uint8_t* b_scales, void* C,
                                       adahop_dtype_t out_dt, int64_t ldc, int64_t M, int64_t N,
                                       int64_t K, void* ws, size_t ws_bytes,
                                       adahop_stream_t stream) {
  if (!a_codes || !a_scales || !b_codes || !b_scales || !C || !ws) return ADAHOP_E_INVALID_ARG;
  if (M <= 0 || N <= 0 || K <= 0 || K % 32) return ADAHOP_E_SHAPE;
  if (ldc < N || !aligned16(a_codes) || !aligned16(b_codes) || !aligned16(C))
    return ADAHOP_E_INVALID_ARG;
  if (ws_bytes < adahop_debug_gemm_workspace_bytes(M, N, K) ||
      (reinterpret_cast<uintptr_t>(ws) & 255))
    return ADAHOP_E_WORKSPACE;
  DevInfo dev;
  adahop_status_t st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  Carver c;
  uint8_t* w = static_cast<uint8_t*>(ws);
  uint8_t* sfa = w + c.take(size_t(sf_bytes(M, K)));
  uint8_t* sfb = w + c.take(size_t(sf_bytes(N, K)));
  ADAHOP_LAUNCH(cudaMemsetAsync(sfa, 0, size_t(sf_bytes(M, K)), cs));
  ADAHOP_LAUNCH(cudaMemsetAsync(sfb, 0, size_t(sf_bytes(N, K)), cs));
  ADAHOP_LAUNCH(launch_sf_convert(a_scales, M, K, sfa, false, cs));
  ADAHOP_LAUNCH(launch_sf_convert(b_scales, N, K, sfb, false, cs));
  Mxf4GemmArgs ma{a_codes, sfa, b_codes, sfb, C, out_dt == ADAHOP_DT_F32, ldc, M, N, K};
  ADAHOP_LAUNCH(run_gemm_mxf4(ma, dev.sms, cs));
  g_launches = 3;
  return ADAHOP_OK;
}

size_t adahop_debug_sf_bytes(int64_t rows, int64_t K) {
  if (rows <= 0 || K <= 0 || K % 32) return 0;
  return size_t(sf_bytes(rows, K));
}

adahop_status_t adahop_debug_gemm_mxf4_tcsf(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes,
                                            const uint8_t* b_sf, void* C, adahop_dtype_t out_dt, int64_t ldc,
                                            int64_t M, int64_t N, int64_t K, adahop_stream_t stream) {
  if (!a_codes || !a_sf || !b_codes || !b_sf || !C) return ADAHOP_E_INVALID_ARG;
  if (M <= 0 || N <= 0 || K <= 0 || K % 32) return ADAHOP_E_SHAPE;
  if (ldc < N || !aligned16(a_codes) || !aligned16(b_codes) || !aligned16(C) || !aligned16(a_sf) || !aligned16(b_sf))
    return ADAHOP_E_INVALID_ARG;
  DevInfo dev;
  adahop_status_t st = check_device(&dev);
  if (st != ADAHOP_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  Mxf4GemmArgs ma{a_codes, a_sf, b_codes, b_sf, C, out_dt == ADAHOP_DT_F32, ldc, M, N, K};
  ADAHOP_LAUNCH(run_gemm_mxf4(ma, dev.sms, cs));
  g_launches = 1;
  return ADAHOP_OK;
}

adahop_status_t adahop_debug_e2m1(const float* v, int64_t n, uint8_t* codes_hw, uint8_t* codes_sw,
                                  adahop_stream_t stream) {
  if (!v || !codes_hw || !codes_sw || n < 0) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  if (n == 0) return ADAHOP_OK;
  ADAHOP_LAUNCH(launch_e2m1_codes(v, n, codes_hw, codes_sw, reinterpret_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return ADAHOP_OK;
}

adahop_status_t adahop_debug_e2m1_exhaustive(uint64_t lo, uint64_t hi,
                                             unsigned long long* d_mismatches,
                                             uint32_t* d_first_bad, adahop_stream_t stream) {
  if (!d_mismatches || !d_first_bad || hi < lo || hi > (1ull << 32)) return ADAHOP_E_INVALID_ARG;
  adahop_status_t st = check_device(nullptr);
  if (st != ADAHOP_OK) return st;
  ADAHOP_LAUNCH(launch_e2m1_exhaustive(lo, hi, d_mismatches, d_first_bad,
                                       reinterpret_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return ADAHOP_OK;
}

}  // extern "C"
