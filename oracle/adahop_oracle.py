"""AdaHOP oracle (numpy). TEST INFRASTRUCTURE: never imported by the product path.

Notation follows the paper. A GEMM computes C = A·B with A in R^{m x k} and
B in R^{k x n} (eq:inner_hadamard). In stored form:
  * ``A_store`` = A as an M x K array (K contiguous),
  * ``B_store`` = B^T as an N x K array.
OE-Left extracts rows of A_store (rows of A); OE-Right extracts rows of B_store
(columns of B). IHT always runs along K.

Readings of silent / garbled passages are listed in DESIGN.md §"Readings"; each is
referenced below as [R<n>].
"""
from __future__ import annotations

import math
from collections import Counter

import numpy as np

HAD_BLOCK = 32          # P:761 "1D FWHT with block size 32"
OE_K = 64               # P:271 "k = 64"
FOID_PROBE = 64         # P:760 "variance of the first 64 elements"
TAU = 2.0               # P:541 "we use tau = 2.0"
EPS = 1e-8              # P:529 "epsilon is a small constant" [R6: 1e-8, SPEC S:227]

# E2M1 magnitudes indexed by the 3-bit code (exponent 2 bits, mantissa 1 bit).
# OCP MX v1.0 FP4 E2M1 (format named P:18; codebook per SPEC S:139).
E2M1_VALUES = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], dtype=np.float64)

# Strategy names (tab:strategy_summary)
IHT, OE_LEFT, OE_RIGHT, BF16 = "IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT", "BF16"


# ======================================================================================
# Hadamard (P:92-99 eq:inner_hadamard; P:761 block 32)
# ======================================================================================
def hadamard_matrix(b: int = HAD_BLOCK, normalized: bool = True) -> np.ndarray:
    """Sylvester/natural-order Walsh-Hadamard matrix, H[i,j] = (-1)^popcount(i&j).

    P:93 "normalized Walsh-Hadamard matrix H_k ... H_k^T H_k = I". Ordering is not
    stated; natural (Sylvester) order is used [R1]."""
    if b < 1 or (b & (b - 1)):
        raise ValueError("Hadamard size must be a power of two")
    i = np.arange(b)[:, None]
    j = np.arange(b)[None, :]
    parity = np.vectorize(lambda v: bin(int(v)).count("1") & 1)(i & j)
    h = np.where(parity == 1, -1.0, 1.0)
    return h / math.sqrt(b) if normalized else h


def iht_dense(x: np.ndarray, b: int = HAD_BLOCK) -> np.ndarray:
    """Blockwise IHT along the last axis as a dense fp64 matrix multiply.

    For A_store rows this is A·H_k (blockwise); for B_store rows it is (H_k^T B)^T
    since H is symmetric. Returns fp64."""
    x = np.asarray(x, dtype=np.float64)
    r, k = x.shape
    if k % b:
        raise ValueError("K must be a multiple of the Hadamard block")
    h = hadamard_matrix(b)
    return (x.reshape(r, k // b, b) @ h).reshape(r, k)


def fwht_fp32_spec(x: np.ndarray, b: int = HAD_BLOCK) -> np.ndarray:
    """fp32 butterfly specification of the same transform [R2].

    Radix-2 stages with strides 1, 2, 4, ..., b/2; each pair (a at i, c at i+h with
    i & h == 0) becomes (a + c, a - c), computed in IEEE fp32 round-to-nearest; the
    result is multiplied by RN32(1/sqrt(b)). This is the fp32 tensor that enters the
    quantiser, used for the bit-exact code/scale contract (north star)."""
    y = np.array(x, dtype=np.float32, copy=True)
    r, k = y.shape
    if k % b:
        raise ValueError("K must be a multiple of the Hadamard block")
    y = y.reshape(r, k // b, b)
    h = 1
    while h < b:
        for i in range(b):
            if i & h:
                continue
            a = y[:, :, i].copy()
            c = y[:, :, i + h].copy()
            y[:, :, i] = a + c
            y[:, :, i + h] = a - c
        h *= 2
    inv = np.float32(1.0 / math.sqrt(b))
    return (y * inv).reshape(r, k).astype(np.float32)


# ======================================================================================
# MXFP4 quantiser (format: "MXFP4"; OCP-MX reference quantiser, north star)
# ======================================================================================
def mx_scale_exponent(amax: np.ndarray) -> np.ndarray:
    """Shared E8M0 exponent per block: e = floor(log2(amax)) - emax(E2M1) with emax=2,
    clamped to [-127, 127]; an all-zero block gets e = 0 [R3]."""
    amax = np.asarray(amax, dtype=np.float64)
    e = np.zeros(amax.shape, dtype=np.int64)
    nz = amax > 0
    m, ex = np.frexp(amax[nz])          # amax = m * 2^ex, m in [0.5, 1)
    e[nz] = (ex - 1) - 2                # floor(log2 amax) = ex - 1
    return np.clip(e, -127, 127)


def e2m1_code(v: np.ndarray) -> np.ndarray:
    """Round v (already divided by the block scale) to the E2M1 code.

    Nearest magnitude in {0,.5,1,1.5,2,3,4,6}; |v| >= 6 saturates to 6 (satfinite);
    an exact tie goes to the code whose mantissa bit is 0 (round-half-even) [R4].
    Sign bit (bit 3) = signbit(v), so negative values that round to zero give 0x8."""
    v = np.asarray(v, dtype=np.float64)
    mag = np.abs(v)
    d = np.abs(mag[..., None] - E2M1_VALUES)                  # distance to each code
    best = d.min(axis=-1, keepdims=True)
    cand = d == best                                          # 1 or 2 nearest codes
    # among the nearest, prefer an even code index (mantissa bit 0)
    even_pref = cand & ((np.arange(8) & 1) == 0)
    has_even = even_pref.any(axis=-1, keepdims=True)
    pick = np.where(has_even, even_pref, cand)
    code = np.argmax(pick, axis=-1).astype(np.uint8)
    code = np.where(mag >= 6.0, np.uint8(7), code)
    sign = np.signbit(v).astype(np.uint8) << 3
    return (code | sign).astype(np.uint8)


def quantize_mxfp4(y: np.ndarray, block: int = 32):
    """MXFP4-quantise each row of y along its last axis in blocks of 32.

    Returns (codes uint8 [R, K] with 4-bit values, scale_bytes uint8 [R, K/32] holding
    the biased E8M0 exponent e + 127). Q(.) of P:82-84 / P:95."""
    y = np.asarray(y)
    r, k = y.shape
    if k % block:
        raise ValueError("K must be a multiple of 32")
    codes = np.empty((r, k), dtype=np.uint8)
    scales = np.empty((r, k // block), dtype=np.uint8)
    step = max(1, (1 << 20) // max(k, 1))                     # bound temporary memory
    for r0 in range(0, r, step):
        yb = y[r0:r0 + step].astype(np.float64).reshape(-1, k // block, block)
        amax = np.abs(yb).max(axis=-1)
        e = mx_scale_exponent(amax)
        v = yb / np.exp2(e.astype(np.float64))[..., None]    # exact power-of-two division
        codes[r0:r0 + step] = e2m1_code(v).reshape(-1, k)
        scales[r0:r0 + step] = (e + 127).astype(np.uint8)
    return codes, scales


def dequantize_mxfp4(codes: np.ndarray, scale_bytes: np.ndarray, block: int = 32) -> np.ndarray:
    """code value x 2^e, exact in fp64."""
    codes = np.asarray(codes, dtype=np.uint8)
    r, k = codes.shape
    mag = E2M1_VALUES[codes & 7]
    val = np.where(codes & 8, -mag, mag).reshape(r, k // block, block)
    e = scale_bytes.astype(np.int64) - 127
    return (val * np.exp2(e.astype(np.float64))[..., None]).reshape(r, k)


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """Canonical packing: R x K/2 bytes, element 2j in the low nibble."""
    codes = np.asarray(codes, dtype=np.uint8)
    return (codes[:, 0::2] | (codes[:, 1::2] << 4)).astype(np.uint8)


def unpack_codes(packed: np.ndarray) -> np.ndarray:
    packed = np.asarray(packed, dtype=np.uint8)
    r, kh = packed.shape
    out = np.empty((r, 2 * kh), dtype=np.uint8)
    out[:, 0::2] = packed & 0xF
    out[:, 1::2] = packed >> 4
    return out


def round_bf16(x: np.ndarray) -> np.ndarray:
    """IEEE round-to-nearest-even of float32 values to bf16 (returned as float64)."""
    x32 = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    bits = x32.view(np.uint32).astype(np.uint64)
    keep = bits >> 16
    rem = bits & 0xFFFF
    up = (rem > 0x8000) | ((rem == 0x8000) & ((keep & 1) == 1))
    keep = keep + up.astype(np.uint64)
    return (keep << 16).astype(np.uint32).view(np.float32).astype(np.float64).reshape(x32.shape)


# ======================================================================================
# FOID + OE split (P:350, P:760 stage 1; P:271-283 eq:oe_left / eq:oe_right)
# ======================================================================================
def foid_keys(store: np.ndarray, probe: int = FOID_PROBE) -> np.ndarray:
    """Variance of the first min(probe, K) elements of each stored row.

    P:760 "computing the variance of the first 64 elements along each row (or column)".
    Population variance, signed values, fp64, accumulated sequentially j = 0..p-1 with
    separate multiply and add (no FMA) [R5] so the key is bit-reproducible."""
    r, k = np.shape(store)
    p = min(probe, k)
    x = np.asarray(np.asarray(store)[:, :p], dtype=np.float64)    # only the probe is read
    s = np.zeros(r, dtype=np.float64)
    for j in range(p):
        s = s + x[:, j]
    mu = s / p
    v = np.zeros(r, dtype=np.float64)
    for j in range(p):
        d = x[:, j] - mu
        v = v + d * d
    return v / p


def foid_indices(store: np.ndarray, k: int = OE_K, probe: int = FOID_PROBE) -> np.ndarray:
    """Top-k rows of the stored operand by FOID key; ties -> lower index [R5];
    k clamped to the row count; returned sorted ascending."""
    keys = foid_keys(store, probe)
    r = keys.shape[0]
    k = max(0, min(int(k), r))
    order = sorted(range(r), key=lambda i: (-keys[i], i))    # brute-force full sort
    return np.array(sorted(order[:k]), dtype=np.int64)


def oe_split(store: np.ndarray, idx: np.ndarray):
    """Residual = input with rows idx set to +0; outlier slice = those rows verbatim
    ("A = A_res + A_out", "corresponding entries in the residual tensor are
    zeroed out")."""
    store = np.asarray(store)
    res = store.copy()
    res[idx, :] = 0.0
    return res, store[idx, :].copy()


# ======================================================================================
# Strategy table (tab:strategy_summary P:305-326, rules P:262-301)
# ======================================================================================
_TABLE = {
    ("C", "N"): IHT, ("N", "N"): IHT, ("R", "N"): OE_LEFT, ("R", "C"): OE_RIGHT,
    ("N", "C"): OE_RIGHT, ("C", "R"): IHT, ("R", "R"): OE_LEFT, ("N", "R"): IHT,
}


def strategy_for_pair(left: str, right: str, level: int = 1) -> str:
    """P:314-323; CC -> OE-Right (Lv1) / BF16 (Lv2) per P:299-300."""
    if (left, right) == ("C", "C"):
        return OE_RIGHT if level == 1 else BF16
    return _TABLE[(left, right)]


# ======================================================================================
# Calibration (App A; §5.1)
# ======================================================================================
def cv_row_col(t: np.ndarray, eps: float = EPS):
    """CV_row = (1/m) sum_i std(T_i,:)/(mean|T_i,:| + eps) and CV_col analogue.
    Population std [R6]."""
    t = np.asarray(t, dtype=np.float64)
    cv_row = float(np.mean(np.std(t, axis=1) / (np.mean(np.abs(t), axis=1) + eps)))
    cv_col = float(np.mean(np.std(t, axis=0) / (np.mean(np.abs(t), axis=0) + eps)))
    return cv_row, cv_col


def classify(t: np.ndarray, tau: float = TAU, eps: float = EPS) -> str:
    """Row if CV_col > tau, Column if CV_row > tau, else None.

    Reading [R7]: the printed /sqrt(dim) normaliser bounds the statistic
    below 1 so tau = 2 could never fire; the raw CV is compared with tau. When both
    exceed tau the larger wins; an exact tie goes to Row."""
    cv_row, cv_col = cv_row_col(t, eps)
    row_hit, col_hit = cv_col > tau, cv_row > tau
    if row_hit and (not col_hit or cv_col >= cv_row):
        return "R"
    if col_hit:
        return "C"
    return "N"


KAPPA = 32.0            # [R16] the factor standing for App. D's ">>"


def outlier_counts(t: np.ndarray, kappa: float = KAPPA):
    """Outlier rows and columns of t (App. D): row i is an outlier row when
    max_j |t_ij| >> median |t|, column j likewise. Reading [R16]: the median over all entries is
    replaced by the mean |t| = sum |t| / (m n) (both computed in fp64; for the unimodal bulk the
    two differ by a constant factor that kappa absorbs) and ">>" by kappa = 32.
    Returns (rows, cols)."""
    a = np.abs(np.asarray(t, dtype=np.float64))
    thr = kappa * (a.sum() / a.size)
    return int((a.max(axis=1) > thr).sum()), int((a.max(axis=0) > thr).sum())


def adaptive_k(count: int, k_max: int = OE_K, granule: int = 16) -> int:
    """Per-layer OE k (P:503 names "an adaptive per-layer selection strategy based on per-layer
    outlier severity" as future work; reading [R16]): the OE operand's outlier rows (stored
    orientation) rounded up to the tcgen05 N granule, clamped to [granule, k_max]."""
    return int(min(k_max, max(granule, -(-int(count) // granule) * granule)))


def transpose_pattern(p: str) -> str:
    """pattern(T^T) = swap(R <-> C) [R8] — CV_row(T^T) = CV_col(T)."""
    return {"R": "C", "C": "R", "N": "N"}[p]


def majority_vote(patterns) -> str:
    """Mode of the per-step patterns; tie priority R > C > N [R9]."""
    if len(patterns) == 0:
        raise ValueError("empty calibration record")
    cnt = Counter(patterns)
    best = max(cnt.values())
    for p in ("R", "C", "N"):
        if cnt.get(p, 0) == best:
            return p
    raise AssertionError


# ======================================================================================
# Linear-layer paths (P:72-79 eq:forward / eq:backward_gw / eq:backward_gx)
# ======================================================================================
def path_operands(path: str, x=None, w=None, gy=None):
    """Return (A_store, B_store) for a path, in the stored K-major convention.

    fwd:   Y   = X W^T    A = X (T x d_in),    B = W^T  -> B_store = W
    dgrad: G_X = G_Y W    A = G_Y (T x d_out), B = W    -> B_store = W^T
    wgrad: G_W = G_Y^T X  A = G_Y^T,           B = X    -> B_store = X^T
    """
    if path == "fwd":
        return np.asarray(x), np.asarray(w)
    if path == "dgrad":
        return np.asarray(gy), np.asarray(w).T
    if path == "wgrad":
        return np.asarray(gy).T, np.asarray(x).T
    raise ValueError(path)


def fed_patterns(path: str, pat_x: str, pat_w: str, pat_gy: str):
    """Pattern pair (left A, right B) of a path, detected on the operand as fed [R8]."""
    t = transpose_pattern
    if path == "fwd":
        return pat_x, t(pat_w)           # A = X, B = W^T
    if path == "dgrad":
        return pat_gy, pat_w             # A = G_Y, B = W
    if path == "wgrad":
        return t(pat_gy), pat_x          # A = G_Y^T, B = X
    raise ValueError(path)


# ======================================================================================
# AdaHOP matmul (eq:inner_hadamard P:95, eq:oe_left P:273, eq:oe_right P:280)
# ======================================================================================
def quantize_operand(store: np.ndarray, hadamard: str = "spec", b: int = HAD_BLOCK):
    """IHT + Q on a stored operand (rows along K). hadamard='spec' uses the fp32
    butterfly spec (bit-exact contract), 'dense' the fp64 dense matrix product."""
    if hadamard == "spec":
        y = fwht_fp32_spec(np.asarray(store, dtype=np.float32), b)
    elif hadamard == "dense":
        y = iht_dense(store, b)
    elif hadamard == "none":
        y = np.asarray(store, dtype=np.float64)
    else:
        raise ValueError(hadamard)
    return quantize_mxfp4(y)


def adahop_matmul(a_store, b_store, strategy: str, k: int = OE_K, probe: int = FOID_PROBE,
                  hadamard: str = "spec", return_parts: bool = False):
    """C (M x N, fp64) for one AdaHOP GEMM in stored form.

    IHT:       C = Q(A H) Q(H^T B)
    OE-Left:   C = Q(A_res H) Q(H^T B) + A_out B, A_out = top-k rows of A
    OE-Right:  C = Q(A H) Q(H^T B_res) + A B_out, B_out = top-k cols of B
    BF16:      C = A B in BF16 operands                    (Lv2)
    The outlier (BF16) path uses bf16-rounded operands, accumulated in fp64 [R10]."""
    a_store = np.asarray(a_store, dtype=np.float32)
    b_store = np.asarray(b_store, dtype=np.float32)
    m, kk = a_store.shape
    n, kb = b_store.shape
    if kk != kb:
        raise ValueError("inner dimensions differ")
    parts = {}
    if strategy == BF16:
        c = round_bf16(a_store) @ round_bf16(b_store).T
        return (c, parts) if return_parts else c
    a_res, b_res = a_store, b_store
    idx = np.zeros(0, dtype=np.int64)
    if strategy == OE_LEFT and k > 0:
        idx = foid_indices(a_store, k, probe)
        a_res, a_out = oe_split(a_store, idx)
    elif strategy == OE_RIGHT and k > 0:
        idx = foid_indices(b_store, k, probe)
        b_res, b_out = oe_split(b_store, idx)
    elif strategy not in (IHT, OE_LEFT, OE_RIGHT):
        raise ValueError(strategy)
    qa = quantize_operand(a_res, hadamard)
    qb = quantize_operand(b_res, hadamard)
    c_main = dequantize_mxfp4(*qa) @ dequantize_mxfp4(*qb).T
    c = c_main.copy()
    if strategy == OE_LEFT and len(idx):
        c_out = round_bf16(a_out) @ round_bf16(b_store).T          # k x N
        c[idx, :] += c_out
        parts["c_out"] = c_out
    elif strategy == OE_RIGHT and len(idx):
        c_out = round_bf16(a_store) @ round_bf16(b_out).T          # M x k
        c[:, idx] += c_out
        parts["c_out"] = c_out
    parts.update(idx=idx, qa=qa, qb=qb, c_main=c_main)
    return (c, parts) if return_parts else c


def linear(path: str, strategy: str, x=None, w=None, gy=None, **kw):
    """One AdaHOP linear path via adahop_matmul on the stored operands."""
    a_store, b_store = path_operands(path, x=x, w=w, gy=gy)
    return adahop_matmul(a_store, b_store, strategy, **kw)


# ======================================================================================
# Analysis helpers (P:604-607 outlier factor gamma; P:161-163 MSE improvement)
# ======================================================================================
def gamma(a: np.ndarray) -> float:
    """gamma(A) = m n max|a_ij|^2 / ||A||_F^2."""
    a = np.asarray(a, dtype=np.float64)
    return float(a.size * np.max(np.abs(a)) ** 2 / np.sum(a * a))


def sampled_entries(a_store, b_store, strategy, rows, cols, k=OE_K, probe=FOID_PROBE):
    """Oracle values C[rows[i], cols[i]] at full size without forming C: FOID runs on the
    full probe, only the needed rows of A_store / B_store are quantised."""
    a_store = np.asarray(a_store, dtype=np.float32)
    b_store = np.asarray(b_store, dtype=np.float32)
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    if strategy == BF16:
        ra = round_bf16(a_store[rows])
        rb = round_bf16(b_store[cols])
        return np.sum(ra * rb, axis=1)
    sa = np.zeros(0, np.int64)
    sb = np.zeros(0, np.int64)
    if strategy == OE_LEFT and k > 0:
        sa = foid_indices(a_store, k, probe)
    if strategy == OE_RIGHT and k > 0:
        sb = foid_indices(b_store, k, probe)
    ur, inv_r = np.unique(rows, return_inverse=True)
    uc, inv_c = np.unique(cols, return_inverse=True)
    ar = a_store[ur].copy()
    bc = b_store[uc].copy()
    ar[np.isin(ur, sa)] = 0.0
    bc[np.isin(uc, sb)] = 0.0
    da = dequantize_mxfp4(*quantize_operand(ar))
    db = dequantize_mxfp4(*quantize_operand(bc))
    out = np.sum(da[inv_r] * db[inv_c], axis=1)
    if len(sa):
        hit = np.isin(rows, sa)
        out[hit] += np.sum(round_bf16(a_store[rows[hit]]) * round_bf16(b_store[cols[hit]]), axis=1)
    if len(sb):
        hit = np.isin(cols, sb)
        out[hit] += np.sum(round_bf16(a_store[rows[hit]]) * round_bf16(b_store[cols[hit]]), axis=1)
    return out
