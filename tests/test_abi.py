"""CPU tests of the C ABI boundary: the library loads, exports every symbol declared in
include/adahop.h, and the pure host functions / host-side validation behave (no compute
calls — there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

import oracle as O
from conftest import ROOT, golden

ah = pytest.importorskip("paper_2604_02525_b200")
from paper_2604_02525_b200 import _lib  # noqa: E402


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "adahop.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adahop_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    names = _declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), n
        assert n in _lib.SIGNATURES, f"{n} declared in adahop.h but not bound in _lib.py"
    assert set(_lib.SIGNATURES) == set(names)


def test_abi_version_and_defaults():
    assert _lib.lib.adahop_abi_version() == 2
    p = _lib.Params(0, 0, 0, 0, 0.0, 0.0)
    _lib.lib.adahop_default_params(C.byref(p))
    assert (p.had_block, p.oe_k, p.foid_probe, p.level) == (32, 64, 64, 1)
    assert abs(p.tau - 2.0) < 1e-7 and abs(p.eps - 1e-8) < 1e-12


def test_strategy_table_matches_golden_and_oracle():
    for left, right, level, strat in golden("strategy_table.txt"):
        assert ah.strategy_for_pair(left, right, int(level)) == strat
        assert O.strategy_for_pair(left, right, int(level)) == strat


def test_majority_vote_and_classify_cv_match_oracle():
    for seq in (["R"] * 30, ["R"] * 16 + ["N"] * 14, ["R"] * 15 + ["C"] * 15, ["C"] * 3 + ["N"] * 3,
                ["N"] * 5 + ["C"] * 4 + ["R"] * 4):
        assert ah.majority_vote(seq) == O.majority_vote(seq)
    # an empty or invalid record is an input error on both sides (oracle: ValueError)
    for bad in ([], ["R", "X"]):
        with pytest.raises(ValueError):
            ah.majority_vote(bad)
    assert _lib.lib.adahop_majority_vote(None, 3) == -1
    arr = (C.c_int32 * 2)(1, 7)
    assert _lib.lib.adahop_majority_vote(arr, 2) == -1
    # the library's decision on the oracle's CVs == the oracle's decision, on the closed-form
    # matrices of test_oracle_pins (both above tau each way, exact tie, one side only, neither)
    import numpy as np
    ident = np.eye(16)
    t = np.eye(16)
    t[0, 1:4] = 1.0
    wide = np.zeros((4, 64))
    wide[np.arange(4), np.arange(4) * 16] = 1.0
    for m in (ident, t, t.T, wide, wide.T, np.tile(np.eye(4), (4, 1)), np.full((8, 8), 2.0)):
        assert ah.classify_cv(*O.cv_row_col(m)) == O.classify(m)
    # threshold boundary: strictly greater than tau
    assert ah.classify_cv(2.0, 2.0) == "N"
    assert ah.classify_cv(2.0000001, 2.0) == "C"


def test_status_strings():
    for s in range(7):
        assert _lib.lib.adahop_status_string(s)
    assert b"shape" in _lib.lib.adahop_status_string(2)


def test_host_validation_without_device():
    p = _lib.Params()
    f = _lib.lib
    # null pointers -> invalid argument (checked before any device query)
    assert f.adahop_gemm(None, 0, 64, None, 0, 64, None, 1, 64, 64, 64, 64, 0, C.byref(p), None, 0, None) == 1
    # no device in this container -> the library reports it instead of falling back to the CPU
    buf = (C.c_uint8 * 4096)()
    ptr = C.cast(buf, C.c_void_p)
    st = f.adahop_gemm(ptr, 0, 64, ptr, 0, 64, ptr, 1, 64, 64, 64, 64, 0, C.byref(p), ptr, 4096, None)
    assert st in (6, 4)          # E_NO_DEVICE (or E_WORKSPACE if a device exists)
    # K % 32 != 0 -> shape error before anything else
    assert f.adahop_gemm(ptr, 0, 64, ptr, 0, 64, ptr, 1, 64, 64, 64, 48, 0, C.byref(p), ptr, 4096, None) == 2
    # had_block != 32 -> unsupported
    q = _lib.Params(had_block=16)
    assert f.adahop_gemm(ptr, 0, 64, ptr, 0, 64, ptr, 1, 64, 64, 64, 64, 0, C.byref(q), ptr, 4096, None) == 3
    # the multi-rank decision entry point validates before touching the device
    assert f.adahop_classify_sums(None, 64, 64, C.byref(p), None, None) == 1
    assert f.adahop_classify_sums(ptr, 0, 64, C.byref(p), ptr, None) == 2
    # wgrad needs T % 32 == 0
    assert f.adahop_linear_wgrad(ptr, ptr, ptr, 1, 48, 64, 64, 0, C.byref(p), ptr, 4096, None) == 2
    # batched calibration: empty / null / bad shapes are rejected before the device query
    rows = (C.c_int64 * 2)(64, 64)
    cols = (C.c_int64 * 2)(64, 0)
    ts = (C.c_void_p * 2)(ptr.value, ptr.value)
    assert f.adahop_calibrate_batch(0, ts, 0, rows, cols, rows, C.byref(p), ptr, 4096, ptr, ptr, None) == 1
    assert f.adahop_calibrate_batch(2, None, 0, rows, cols, rows, C.byref(p), ptr, 4096, ptr, ptr, None) == 1
    assert f.adahop_calibrate_batch(2, ts, 0, rows, cols, rows, C.byref(p), ptr, 4096, ptr, ptr, None) == 2
    assert f.adahop_calibrate_batch_workspace_bytes(2, rows, cols) == 0        # a zero-column tensor
    assert f.adahop_calibrate_batch_outliers(2, rows, cols, ptr, 4096, 32.0, ptr, None) == 2
    assert f.adahop_calibrate_batch_outliers(1, rows, rows, ptr, 4096, 0.0, ptr, None) == 1   # kappa must be > 0
    # the GEMM-alone debug entry point: K % 32 and alignment checks before the device
    assert f.adahop_debug_gemm_mxf4_tcsf(ptr, ptr, ptr, ptr, ptr, 1, 64, 64, 64, 48, None) == 2
    assert f.adahop_debug_sf_bytes(128, 48) == 0 and f.adahop_debug_sf_bytes(128, 256) > 0


def test_workspace_sizes_are_host_computable():
    p = _lib.Params()
    n_iht = ah.workspace_bytes("fwd", 16384, 2048, 2048, "IHT", p)
    n_oe = ah.workspace_bytes("fwd", 16384, 2048, 2048, "OE_RIGHT_IHT", p)
    # FP4 codes + scales of both operands at least
    assert n_iht >= (16384 + 2048) * 2048 // 2 + (16384 + 2048) * 2048 // 32
    assert n_oe > n_iht
    assert ah.workspace_bytes("fwd", 16384, 2048, 2048, "BF16", p) <= 512
