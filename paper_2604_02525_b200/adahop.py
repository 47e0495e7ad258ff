"""Python binding of the AdaHOP C ABI (include/adahop.h) over torch tensors.

Argument marshalling only: every arithmetic step runs in libadahop.so's sm_100a kernels.
PyTorch provides device memory (the caching allocator), the current CUDA stream and,
in ``dist.py``, the process group.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import AdahopError, Params, check, lib

IHT, OE_LEFT_IHT, OE_RIGHT_IHT, BF16 = 0, 1, 2, 3
STRATEGY = {"IHT": IHT, "OE_LEFT_IHT": OE_LEFT_IHT, "OE_RIGHT_IHT": OE_RIGHT_IHT, "BF16": BF16}
STRATEGY_NAME = {v: k for k, v in STRATEGY.items()}
PAT = {"N": 0, "R": 1, "C": 2}
PAT_NAME = {0: "N", 1: "R", 2: "C"}
PATH = {"fwd": 0, "dgrad": 1, "wgrad": 2}
DT_BF16, DT_F32 = 0, 1

__all__ = [
    "AdahopError", "Params", "IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT", "BF16", "STRATEGY", "strategy_for_pair",
    "majority_vote", "classify_cv", "stats", "classify", "calibrate", "gemm", "linear",
    "linear_fwd", "linear_dgrad", "linear_wgrad", "workspace_bytes", "debug_iht_quant", "debug_quant_dual",
    "debug_foid", "debug_gemm_mxf4", "debug_e2m1", "debug_e2m1_exhaustive", "last_launch_count",
    "Workspace", "StageEvents", "linear_layer", "layer_workspace_bytes", "calibrate_async",
    "calibrate_workspace_bytes", "classify_sums", "LinearContext", "linear_forward", "linear_backward",
    "split_workspace_bytes", "linear_ctx_bytes", "layer_strategies", "debug_sf_bytes", "debug_gemm_mxf4_tcsf",
    "calibrate_batch_async", "calibrate_batch_workspace_bytes", "calibrate_batch_outliers_async", "KAPPA",
]


def _strategy(s) -> int:
    return STRATEGY[s] if isinstance(s, str) else int(s)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return DT_BF16
    if t.dtype == torch.float32:
        return DT_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


# ------------------------------------------------------------------------- host helpers
def strategy_for_pair(left: str, right: str, level: int = 1) -> str:
    return STRATEGY_NAME[lib.adahop_strategy_for_pair(PAT[left], PAT[right], level)]


def layer_strategies(pat_x: str, pat_w: str, pat_gy: str, level: int = 1):
    """(strategies (fwd, dgrad, wgrad), fed pairs ('XY' strings)) of one linear from the calibrated
    patterns of X, W, G_Y as stored (adahop_layer_strategies)."""
    out = (C.c_int32 * 3)()
    fed = (C.c_int32 * 6)()
    if lib.adahop_layer_strategies(PAT[pat_x], PAT[pat_w], PAT[pat_gy], level, out, fed) != 0:
        raise ValueError(f"invalid patterns / level {(pat_x, pat_w, pat_gy, level)}")
    return (tuple(STRATEGY_NAME[v] for v in out),
            tuple(PAT_NAME[fed[2 * i]] + PAT_NAME[fed[2 * i + 1]] for i in range(3)))


def majority_vote(patterns) -> str:
    """Mode of the per-step patterns (ties R > C > N); ValueError for an empty record."""
    arr = (C.c_int32 * max(1, len(patterns)))(*[PAT.get(p, -1) for p in patterns])
    v = lib.adahop_majority_vote(arr, len(patterns))
    if v < 0:
        raise ValueError(f"invalid calibration record {list(patterns)!r}")
    return PAT_NAME[v]


def classify_cv(cv_row: float, cv_col: float, params: Params | None = None) -> str:
    p = params or Params()
    return PAT_NAME[lib.adahop_classify_cv(cv_row, cv_col, C.byref(p))]


def last_launch_count() -> int:
    return lib.adahop_last_launch_count()


class Workspace:
    """Caller-owned scratch (grown on demand; pointer stable once large enough)."""

    def __init__(self, nbytes: int = 0, device=None):
        self.buf = None
        if nbytes:
            self.ensure(nbytes, device)

    def ensure(self, nbytes: int, device=None) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8,
                                   device=device or torch.cuda.current_device())
        return self.buf


_default_ws: dict = {}


def _ws(nbytes: int, ws: Workspace | None, device) -> torch.Tensor:
    if ws is None:
        ws = _default_ws.setdefault(str(device), Workspace())
    return ws.ensure(nbytes, device)


# ------------------------------------------------------------------------- calibration
def _check_rowmajor(t: torch.Tensor) -> None:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("expected a 2-D tensor with unit column stride (row-major rows)")


def stats(t: torch.Tensor):
    """Per-row and per-column {sum x, sum x^2, sum |x|, max |x|} (fp64) of a 2-D tensor."""
    _check_rowmajor(t)
    rows, cols = t.shape
    rs = torch.empty((rows, 4), dtype=torch.float64, device=t.device)
    cs = torch.empty((cols, 4), dtype=torch.float64, device=t.device)
    n = lib.adahop_stats_workspace_bytes(rows, cols)
    w = torch.empty(n, dtype=torch.uint8, device=t.device)
    check("adahop_stats", lib.adahop_stats(_ptr(t), _dt(t), rows, cols, t.stride(0), _ptr(rs), _ptr(cs),
                                           _ptr(w), n, _stream()))
    return rs, cs


def classify(row_stats, col_stats, row_len: int, col_count: int, params: Params | None = None):
    """adahop_classify: cv (device, 4 doubles: row-CV sum, column-CV sum, CV_row, CV_col) and the
    single-rank pattern (device uint8)."""
    p = params or Params()
    dev = row_stats.device
    cv = torch.empty(4, dtype=torch.float64, device=dev)
    pat = torch.empty(1, dtype=torch.uint8, device=dev)
    rows = row_stats.shape[0]
    cols = col_stats.shape[0]
    assert row_len == cols
    check("adahop_classify", lib.adahop_classify(_ptr(row_stats), rows, _ptr(col_stats), cols, col_count,
                                                 C.byref(p), _ptr(cv), _ptr(pat), _stream()))
    return cv, pat


def classify_sums(cv: torch.Tensor, rows_global: int, cols: int, params: Params | None = None):
    """adahop_classify_sums: the App. A decision from the all-reduced CV sums cv[0], cv[1] (device,
    4 doubles, updated in place: cv[2] = CV_row, cv[3] = CV_col); returns the pattern (device uint8)."""
    p = params or Params()
    assert cv.dtype == torch.float64 and cv.numel() >= 4 and cv.is_contiguous()
    pat = torch.empty(1, dtype=torch.uint8, device=cv.device)
    check("adahop_classify_sums", lib.adahop_classify_sums(_ptr(cv), rows_global, cols, C.byref(p), _ptr(pat),
                                                           _stream()))
    return pat


def calibrate(t: torch.Tensor, params: Params | None = None):
    """One calibration step of one tensor (App. A): returns (pattern 'R'|'C'|'N', cv_row, cv_col)."""
    p = params or Params()
    _check_rowmajor(t)
    rows, cols = t.shape
    n = lib.adahop_calibrate_workspace_bytes(rows, cols)
    w = torch.empty(n, dtype=torch.uint8, device=t.device)
    cv = torch.empty(4, dtype=torch.float64, device=t.device)
    pat = torch.empty(1, dtype=torch.uint8, device=t.device)
    check("adahop_calibrate", lib.adahop_calibrate(_ptr(t), _dt(t), rows, cols, t.stride(0), C.byref(p),
                                                   _ptr(w), n, _ptr(cv), _ptr(pat), _stream()))
    cvh = cv.cpu().tolist()
    return PAT_NAME[int(pat.item())], cvh[2], cvh[3]


def calibrate_async(t: torch.Tensor, ws: torch.Tensor, cv: torch.Tensor, pat: torch.Tensor,
                    params: Params | None = None) -> None:
    """adahop_calibrate without the host read-back (graph-capturable): cv (4 fp64) receives the
    row / column CV sums and CV_row, CV_col, and pat (1 uint8) the pattern code, both on the
    device. ws must hold calibrate_workspace_bytes(rows, cols) bytes."""
    p = params or Params()
    _check_rowmajor(t)
    assert cv.dtype == torch.float64 and cv.numel() >= 4 and cv.is_contiguous()
    rows, cols = t.shape
    check("adahop_calibrate", lib.adahop_calibrate(_ptr(t), _dt(t), rows, cols, t.stride(0), C.byref(p),
                                                   _ptr(ws), ws.numel(), _ptr(cv), _ptr(pat), _stream()))


def calibrate_batch_workspace_bytes(shapes) -> int:
    """Workspace of calibrate_batch_async for tensors of the given (rows, cols) shapes."""
    n = len(shapes)
    rows = (C.c_int64 * n)(*[int(r) for r, _ in shapes])
    cols = (C.c_int64 * n)(*[int(c) for _, c in shapes])
    return int(lib.adahop_calibrate_batch_workspace_bytes(n, rows, cols))


def calibrate_batch_async(tensors, ws: torch.Tensor, cv: torch.Tensor, pat: torch.Tensor,
                          params: Params | None = None) -> None:
    """adahop_calibrate_batch: one calibration step of every tensor in `tensors` (same dtype), three
    launches per 32 tensors, graph-capturable; cv [n, 4] fp64 and pat [n] uint8 receive what n
    calibrate_async calls would write."""
    p = params or Params()
    n = len(tensors)
    for t in tensors:
        _check_rowmajor(t)
        assert t.dtype == tensors[0].dtype
    assert cv.dtype == torch.float64 and cv.is_contiguous() and cv.numel() >= 4 * n
    assert pat.dtype == torch.uint8 and pat.numel() >= n
    ptrs = (C.c_void_p * n)(*[t.data_ptr() for t in tensors])
    rows = (C.c_int64 * n)(*[t.shape[0] for t in tensors])
    cols = (C.c_int64 * n)(*[t.shape[1] for t in tensors])
    ld = (C.c_int64 * n)(*[t.stride(0) for t in tensors])
    check("adahop_calibrate_batch", lib.adahop_calibrate_batch(n, ptrs, _dt(tensors[0]), rows, cols, ld, C.byref(p),
                                                               _ptr(ws), ws.numel(), _ptr(cv), _ptr(pat), _stream()))


KAPPA = 32.0   # DESIGN R16: the factor standing for App. D's ">>"


def calibrate_batch_outliers_async(shapes, ws: torch.Tensor, counts: torch.Tensor, kappa: float = KAPPA) -> None:
    """adahop_calibrate_batch_outliers after calibrate_batch_async with the same shapes and ws: counts
    [n, 2] int32 receives each tensor's outlier rows and columns (DESIGN R16)."""
    n = len(shapes)
    assert counts.dtype == torch.int32 and counts.is_contiguous() and counts.numel() >= 2 * n
    rows = (C.c_int64 * n)(*[int(r) for r, _ in shapes])
    cols = (C.c_int64 * n)(*[int(c) for _, c in shapes])
    check("adahop_calibrate_batch_outliers",
          lib.adahop_calibrate_batch_outliers(n, rows, cols, _ptr(ws), ws.numel(), float(kappa), _ptr(counts),
                                              _stream()))


def calibrate_workspace_bytes(rows: int, cols: int) -> int:
    return int(lib.adahop_calibrate_workspace_bytes(rows, cols))


# ------------------------------------------------------------------------- hot path
def gemm(a, a_kstrided: bool, b, b_kstrided: bool, M: int, N: int, K: int, strategy,
         params: Params | None = None, out: torch.Tensor | None = None,
         out_dtype=torch.bfloat16, ws: Workspace | None = None) -> torch.Tensor:
    """C = A_store · B_store^T under `strategy` (stored-form GEMM of include/adahop.h)."""
    p = params or Params()
    s = _strategy(strategy)
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=a.device)
    lda = a.stride(0)
    ldb = b.stride(0)
    n = lib.adahop_gemm_workspace_bytes(M, N, K, s, C.byref(p))
    w = _ws(n, ws, a.device)
    check("adahop_gemm", lib.adahop_gemm(_ptr(a), int(a_kstrided), lda, _ptr(b), int(b_kstrided), ldb,
                                         _ptr(out), _dt(out), out.stride(0), M, N, K, s, C.byref(p),
                                         _ptr(w), w.numel(), _stream()))
    return out


def workspace_bytes(path: str, T: int, d_in: int, d_out: int, strategy, params: Params | None = None) -> int:
    p = params or Params()
    return lib.adahop_workspace_bytes(PATH[path], T, d_in, d_out, _strategy(strategy), C.byref(p))


def _linear(fn, path, a, b, T, d_in, d_out, shape, strategy, params, out, out_dtype, ws):
    p = params or Params()
    s = _strategy(strategy)
    assert a.is_contiguous() and b.is_contiguous() and a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    if out is None:
        out = torch.empty(shape, dtype=out_dtype, device=a.device)
    n = lib.adahop_workspace_bytes(PATH[path], T, d_in, d_out, s, C.byref(p))
    w = _ws(n, ws, a.device)
    check(fn.__name__, fn(_ptr(a), _ptr(b), _ptr(out), _dt(out), T, d_in, d_out, s, C.byref(p), _ptr(w),
                          w.numel(), _stream()))
    return out


def linear_fwd(x, w, strategy, params=None, out=None, out_dtype=torch.bfloat16, ws=None):
    """Y = X W^T (eq:forward P:75). X: T x d_in, W: d_out x d_in (bf16)."""
    T, d_in = x.shape
    d_out = w.shape[0]
    return _linear(lib.adahop_linear_fwd, "fwd", x, w, T, d_in, d_out, (T, d_out), strategy, params,
                   out, out_dtype, ws)


def linear_dgrad(gy, w, strategy, params=None, out=None, out_dtype=torch.bfloat16, ws=None):
    """G_X = G_Y W (eq:backward_gx P:77). G_Y: T x d_out, W: d_out x d_in."""
    T, d_out = gy.shape
    d_in = w.shape[1]
    return _linear(lib.adahop_linear_dgrad, "dgrad", gy, w, T, d_in, d_out, (T, d_in), strategy, params,
                   out, out_dtype, ws)


def linear_wgrad(gy, x, strategy, params=None, out=None, out_dtype=torch.float32, ws=None):
    """G_W = G_Y^T X (eq:backward_gw P:76). G_Y: T x d_out, X: T x d_in."""
    T, d_out = gy.shape
    d_in = x.shape[1]
    return _linear(lib.adahop_linear_wgrad, "wgrad", gy, x, T, d_in, d_out, (d_out, d_in), strategy, params,
                   out, out_dtype, ws)


def linear(path: str, strategy, x=None, w=None, gy=None, **kw):
    if path == "fwd":
        return linear_fwd(x, w, strategy, **kw)
    if path == "dgrad":
        return linear_dgrad(gy, w, strategy, **kw)
    if path == "wgrad":
        return linear_wgrad(gy, x, strategy, **kw)
    raise ValueError(path)


# ------------------------------------------------------------------------- debug entry points
def debug_iht_quant(x: torch.Tensor, k_strided: bool = False, zero_rows=None, want_had: bool = False):
    """Production IHT+quant kernel on a stored operand; canonical codes/scales (+ fp32 Hadamard)."""
    if k_strided:
        K, R = x.shape
    else:
        R, K = x.shape
    dev = x.device
    codes = torch.empty((R, K // 2), dtype=torch.uint8, device=dev)
    scales = torch.empty((R, K // 32), dtype=torch.uint8, device=dev)
    had = torch.empty((R, K), dtype=torch.float32, device=dev) if want_had else None
    zr = None
    nz = 0
    if zero_rows is not None and len(zero_rows):
        zr = torch.as_tensor(zero_rows, dtype=torch.int32, device=dev).contiguous()
        nz = zr.numel()
    n = lib.adahop_debug_workspace_bytes(R, K)
    w = torch.empty(n, dtype=torch.uint8, device=dev)
    check("adahop_debug_iht_quant",
          lib.adahop_debug_iht_quant(_ptr(x), _dt(x), R, K, x.stride(0), int(k_strided), _ptr(zr), nz,
                                     _ptr(had), _ptr(codes), _ptr(scales), _ptr(w), n, _stream()))
    return codes, scales, had


def debug_quant_dual(x: torch.Tensor, row_zero=None, col_zero=None, want_slices: bool = False):
    """Dual-orientation IHT+quant of a bf16 [R x C] tensor in one pass: (row codes, row scales,
    col codes, col scales[, row slice, col slice]), canonical layouts."""
    R, C = x.shape
    dev = x.device
    qr = torch.empty((R, C // 2), dtype=torch.uint8, device=dev)
    sr = torch.empty((R, C // 32), dtype=torch.uint8, device=dev)
    qc = torch.empty((C, R // 2), dtype=torch.uint8, device=dev)
    sc = torch.empty((C, R // 32), dtype=torch.uint8, device=dev)

    def idx(z):
        if z is None or len(z) == 0:
            return None, 0
        t = torch.as_tensor(z, dtype=torch.int32, device=dev).contiguous()
        return t, t.numel()

    rz, nr = idx(row_zero)
    cz, nc = idx(col_zero)
    slr = torch.zeros((nr, C), dtype=torch.bfloat16, device=dev) if want_slices and nr else None
    slc = torch.zeros((nc, R), dtype=torch.bfloat16, device=dev) if want_slices and nc else None
    n = lib.adahop_debug_workspace_bytes(R, C) + lib.adahop_debug_workspace_bytes(C, R)
    w = torch.empty(n, dtype=torch.uint8, device=dev)
    check("adahop_debug_quant_dual",
          lib.adahop_debug_quant_dual(_ptr(x), _dt(x), R, C, x.stride(0), _ptr(rz), nr, _ptr(cz), nc, _ptr(qr),
                                      _ptr(sr), _ptr(qc), _ptr(sc), _ptr(slr), _ptr(slc), _ptr(w), n, _stream()))
    if want_slices:
        return qr, sr, qc, sc, slr, slc
    return qr, sr, qc, sc


def debug_foid(x: torch.Tensor, k: int, probe: int = 64, k_strided: bool = False):
    if k_strided:
        K, R = x.shape
    else:
        R, K = x.shape
    dev = x.device
    kk = min(k, R)
    idx = torch.empty(kk, dtype=torch.int32, device=dev)
    keys = torch.empty(R, dtype=torch.float64, device=dev)
    n = lib.adahop_debug_workspace_bytes(R, K)
    w = torch.empty(n, dtype=torch.uint8, device=dev)
    check("adahop_debug_foid", lib.adahop_debug_foid(_ptr(x), _dt(x), R, K, x.stride(0), int(k_strided), k,
                                                     probe, _ptr(idx), _ptr(keys), _ptr(w), n, _stream()))
    return idx, keys


def debug_gemm_mxf4(a_codes, a_scales, b_codes, b_scales, out_dtype=torch.float32):
    M, Kh = a_codes.shape
    N = b_codes.shape[0]
    K = 2 * Kh
    dev = a_codes.device
    out = torch.empty((M, N), dtype=out_dtype, device=dev)
    n = lib.adahop_debug_gemm_workspace_bytes(M, N, K)
    w = torch.empty(n, dtype=torch.uint8, device=dev)
    check("adahop_debug_gemm_mxf4",
          lib.adahop_debug_gemm_mxf4(_ptr(a_codes), _ptr(a_scales), _ptr(b_codes), _ptr(b_scales), _ptr(out),
                                     _dt(out), out.stride(0), M, N, K, _ptr(w), n, _stream()))
    return out


def debug_sf_bytes(rows: int, K: int) -> int:
    return int(lib.adahop_debug_sf_bytes(rows, K))


def debug_gemm_mxf4_tcsf(a_codes, a_sf, b_codes, b_sf, out):
    """The MXFP4 GEMM kernel alone: scales already in the tcgen05 layout (debug_sf_bytes each)."""
    M, Kh = a_codes.shape
    N = b_codes.shape[0]
    for t in (a_codes, b_codes, a_sf, b_sf, out):
        assert t.is_cuda and t.is_contiguous()
    assert out.shape == (M, N) and a_sf.numel() >= debug_sf_bytes(M, 2 * Kh) and b_sf.numel() >= debug_sf_bytes(N, 2 * Kh)
    check("adahop_debug_gemm_mxf4_tcsf",
          lib.adahop_debug_gemm_mxf4_tcsf(_ptr(a_codes), _ptr(a_sf), _ptr(b_codes), _ptr(b_sf), _ptr(out), _dt(out),
                                          out.stride(0), M, N, 2 * Kh, _stream()))
    return out


def debug_e2m1(v: torch.Tensor):
    """(hardware codes, software-rule codes) of fp32 values through the quantiser's conversion."""
    v = v.contiguous().float()
    hw = torch.empty(v.numel(), dtype=torch.uint8, device=v.device)
    sw = torch.empty_like(hw)
    check("adahop_debug_e2m1", lib.adahop_debug_e2m1(_ptr(v), v.numel(), _ptr(hw), _ptr(sw), _stream()))
    return hw, sw


def debug_e2m1_exhaustive(lo: int = 0, hi: int = 1 << 32, device=None):
    """Mismatch count and first mismatching fp32 bit pattern between hw and sw conversion."""
    dev = device or torch.cuda.current_device()
    mism = torch.zeros(1, dtype=torch.int64, device=dev)
    first = torch.full((1,), -1, dtype=torch.int32, device=dev)   # 0xFFFFFFFF
    check("adahop_debug_e2m1_exhaustive",
          lib.adahop_debug_e2m1_exhaustive(lo, hi, _ptr(mism), _ptr(first), _stream()))
    return int(mism.item()), int(first.item()) & 0xFFFFFFFF


class StageEvents:
    """Five CUDA events recorded by the library between the hot-path stages of one call
    (FOID | quant | BF16 outlier GEMM | MXFP4 GEMM + fused outlier scatter), mirroring tab:latency
    (P:451-473)."""

    NAMES = ("foid", "quant", "outlier", "gemm_mxf4")

    def __init__(self):
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        for e in self.events:      # materialise the cudaEvent_t handles
            e.record()
        self._arr = (C.c_void_p * 5)(*[e.cuda_event for e in self.events])

    def __enter__(self):
        lib.adahop_set_stage_events(C.cast(self._arr, C.c_void_p))
        return self

    def __exit__(self, *exc):
        lib.adahop_set_stage_events(None)

    def times_ms(self):
        ev = self.events
        return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(self.NAMES)}


def _strats(strategies):
    return (C.c_int32 * 3)(*[_strategy(v) for v in strategies])


def linear_layer(x, w, gy, strategies, params=None, out_dtype=torch.bfloat16, out=None, ws=None,
                 gw_dtype=None):
    """fwd / dgrad / wgrad of one linear in one call (adahop_linear_layer): every input tensor
    is quantised once in both orientations. strategies = (fwd, dgrad, wgrad). Y and G_X are
    written in out_dtype, G_W in gw_dtype (default: out_dtype)."""
    p = params or Params()
    T, d_in = x.shape
    d_out = w.shape[0]
    for t in (x, w, gy):
        assert t.is_contiguous() and t.dtype == torch.bfloat16
    assert tuple(w.shape) == (d_out, d_in) and tuple(gy.shape) == (T, d_out)
    s = _strats(strategies)
    gw_dtype = gw_dtype or out_dtype
    if out is None:
        out = (torch.empty((T, d_out), dtype=out_dtype, device=x.device),
               torch.empty((T, d_in), dtype=out_dtype, device=x.device),
               torch.empty((d_out, d_in), dtype=gw_dtype, device=x.device))
    y, gx, gw = out
    for o, shape, dt in ((y, (T, d_out), y.dtype), (gx, (T, d_in), y.dtype), (gw, (d_out, d_in), gw.dtype)):
        if tuple(o.shape) != shape or not o.is_contiguous() or o.dtype != dt:
            raise ValueError(f"linear_layer outputs must be contiguous tensors of shapes {(T, d_out)}, "
                             f"{(T, d_in)}, {(d_out, d_in)} (Y and G_X of one dtype)")
    n = lib.adahop_layer_workspace_bytes(T, d_in, d_out, s, C.byref(p))
    wbuf = _ws(n, ws, x.device)
    check("adahop_linear_layer",
          lib.adahop_linear_layer(_ptr(x), _ptr(w), _ptr(gy), _ptr(y), _ptr(gx), _ptr(gw), _dt(y), _dt(gw), T, d_in,
                                  d_out, s, C.byref(p), _ptr(wbuf), wbuf.numel(), _stream()))
    return y, gx, gw


def layer_workspace_bytes(T, d_in, d_out, strategies, params=None) -> int:
    p = params or Params()
    return lib.adahop_layer_workspace_bytes(T, d_in, d_out, _strats(strategies), C.byref(p))


class LinearContext:
    """What adahop_linear_forward saves for adahop_linear_backward: the column-layout FP4
    copies of X and W with their OE indices and BF16 outlier slices, in one device buffer; plus a
    reference to X itself only when the wgrad strategy needs all of X in BF16 (wgrad OE-Left or
    the Lv2 BF16 wgrad; adahop_linear_backward_needs_x)."""

    def __init__(self, T, d_in, d_out, strategies, params, device):
        self.shape = (T, d_in, d_out)
        self.strategies = tuple(strategies)
        self.params = params
        s = _strats(strategies)
        n = lib.adahop_linear_ctx_bytes(T, d_in, d_out, s, C.byref(params))
        self.buf = torch.empty(max(n, 256), dtype=torch.uint8, device=device)
        self.needs_x = bool(lib.adahop_linear_backward_needs_x(s, C.byref(params)))
        self.x = None

    @property
    def saved_bytes(self) -> int:
        """Device bytes kept alive between forward and backward for this linear."""
        return self.buf.numel() + (self.x.numel() * self.x.element_size() if self.x is not None else 0)


def linear_ctx_bytes(T, d_in, d_out, strategies, params=None) -> int:
    """Bytes of the context adahop_linear_forward saves for adahop_linear_backward."""
    p = params or Params()
    return lib.adahop_linear_ctx_bytes(T, d_in, d_out, _strats(strategies), C.byref(p))


def split_workspace_bytes(T, d_in, d_out, strategies, params=None) -> int:
    p = params or Params()
    return lib.adahop_linear_split_workspace_bytes(T, d_in, d_out, _strats(strategies), C.byref(p))


def linear_forward(x, w, strategies, params=None, out=None, out_dtype=torch.bfloat16, ws=None, ctx=None):
    """Y = X W^T and the saved context (adahop_linear_forward). Returns (Y, ctx)."""
    p = params or Params()
    T, d_in = x.shape
    d_out = w.shape[0]
    for t in (x, w):
        assert t.is_contiguous() and t.dtype == torch.bfloat16
    if ctx is None or ctx.shape != (T, d_in, d_out) or ctx.strategies != tuple(strategies):
        ctx = LinearContext(T, d_in, d_out, strategies, p, x.device)
    ctx.params = p
    if out is None:
        out = torch.empty((T, d_out), dtype=out_dtype, device=x.device)
    assert tuple(out.shape) == (T, d_out) and out.is_contiguous()
    s = _strats(strategies)
    n = lib.adahop_linear_split_workspace_bytes(T, d_in, d_out, s, C.byref(p))
    wbuf = _ws(n, ws, x.device)
    check("adahop_linear_forward",
          lib.adahop_linear_forward(_ptr(x), _ptr(w), _ptr(out), _dt(out), T, d_in, d_out, s, C.byref(p),
                                    _ptr(ctx.buf), ctx.buf.numel(), _ptr(wbuf), wbuf.numel(), _stream()))
    ctx.x = x if ctx.needs_x else None
    return out, ctx


def linear_backward(gy, w, ctx: LinearContext, out=None, gx_dtype=torch.bfloat16, gw_dtype=torch.float32,
                    ws=None):
    """G_X = G_Y W and G_W = G_Y^T X from the saved context (adahop_linear_backward)."""
    T, d_in, d_out = ctx.shape
    p = ctx.params
    for t in (gy, w):
        assert t.is_contiguous() and t.dtype == torch.bfloat16
    assert tuple(gy.shape) == (T, d_out) and tuple(w.shape) == (d_out, d_in)
    if out is None:
        out = (torch.empty((T, d_in), dtype=gx_dtype, device=gy.device),
               torch.empty((d_out, d_in), dtype=gw_dtype, device=gy.device))
    gx, gw = out
    assert tuple(gx.shape) == (T, d_in) and tuple(gw.shape) == (d_out, d_in)
    assert gx.is_contiguous() and gw.is_contiguous()
    s = _strats(ctx.strategies)
    n = lib.adahop_linear_split_workspace_bytes(T, d_in, d_out, s, C.byref(p))
    wbuf = _ws(n, ws, gy.device)
    check("adahop_linear_backward",
          lib.adahop_linear_backward(_ptr(gy), _ptr(w), _ptr(ctx.x), _ptr(gx), _ptr(gw), _dt(gx), _dt(gw), T, d_in,
                                     d_out, s, C.byref(p), _ptr(ctx.buf), ctx.buf.numel(), _ptr(wbuf),
                                     wbuf.numel(), _stream()))
    return gx, gw
