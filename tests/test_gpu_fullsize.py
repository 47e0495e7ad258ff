"""Full-size GPU parity in the configuration bench.py times: adahop_linear_layer (all three
GEMMs of one linear, dual-orientation quantisation) at T = 16384 tokens on Llama-3.2-1B,
Instella-3B and Llama-3-8B linear shapes (BASELINE configs[1], [2] and [3], including the OE k
sweep 0 / 16 / 64), checked on sampled output entries against the CPU oracle (the oracle forms only
the sampled entries: FOID on the full probe, quantisation of the sampled rows). Also: bf16
outputs equal RN_bf16 of the fp32 outputs bitwise, and a CUDA-graph replay of
the layer call (as bench.py runs it) equals the eager call bitwise.
"""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_02525_b200 as ah  # noqa: E402

DEV = torch.device("cuda:0")
TOL_OUT = 1e-3   # north star: linear outputs within 1e-3 relative Frobenius


def dev_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, torch.bfloat16)


def rel_fro(got, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(np.asarray(got, np.float64) - ref) / max(np.linalg.norm(ref), 1e-300))


def fed_pair(path, px, pw, pg):
    t = {"R": "C", "C": "R", "N": "N"}
    return {"fwd": (px, t[pw]), "dgrad": (pg, pw), "wgrad": (t[pg], px)}[path]


def sampled_check(path, strategy, got, x, w, gy, k, rng, n=2000):
    a_store, b_store = O.path_operands(path, x=x, w=w, gy=gy)
    a_store, b_store = np.ascontiguousarray(a_store), np.ascontiguousarray(b_store)
    rows = rng.integers(0, got.shape[0], n)
    cols = rng.integers(0, got.shape[1], n)
    if strategy in ("OE_LEFT_IHT", "OE_RIGHT_IHT") and k > 0:
        left = strategy == "OE_LEFT_IHT"
        idx = O.foid_indices(a_store if left else b_store, k)
        extra = rng.integers(0, got.shape[1 if left else 0], len(idx))   # every extracted row / column
        if left:
            rows, cols = np.concatenate([rows, idx]), np.concatenate([cols, extra])
        else:
            rows, cols = np.concatenate([rows, extra]), np.concatenate([cols, idx])
    ref = O.sampled_entries(a_store, b_store, strategy, rows, cols, k=k)
    err = rel_fro(got[rows, cols], ref)
    assert err <= TOL_OUT, (path, strategy, k, err)
    return err


@pytest.mark.slow
@pytest.mark.parametrize("model,linear,k,level", [
    ("llama32_1b", "gate", 64, 1),  # configs[1]: X = C, G_Y = C -> fwd CN (IHT), dgrad CN (IHT), wgrad RC (OE-R)
    ("llama32_1b", "k", 64, 1),     # X = C, G_Y = R -> dgrad RN (OE-L), wgrad CC (OE-R, Lv1)
    ("llama3_8b", "k", 0, 1),       # configs[3] k sweep on the 8B kv projection
    ("llama3_8b", "k", 16, 1),
    ("llama3_8b", "k", 64, 1),
    ("llama3_8b", "k", 64, 2),      # AdaHOP-Lv2: the CC wgrad runs in BF16, full size
    ("instella_3b", "down", 64, 1),  # configs[2]: K = 6912 fwd, N = 6912 dgrad / wgrad
])
def test_linear_layer_full_size_sampled(model, linear, k, level):
    spec = {"llama32_1b": synth.LLAMA32_1B, "llama3_8b": synth.LLAMA3_8B, "instella_3b": synth.INSTELLA_3B}[model]
    _, d_in, d_out = next(t for t in spec["linears"] if t[0] == linear)
    px, pg = synth.LLAMA32_1B_LAYER_PATTERNS[linear]
    T = 16384
    x, _ = synth.operand(T, d_in, px, "X", case_id=501)
    w, _ = synth.operand(d_out, d_in, "N", "W", case_id=502)
    gy, _ = synth.operand(T, d_out, pg, "GY", case_id=503)
    strats = tuple(ah.strategy_for_pair(*fed_pair(p, px, "N", pg), level) for p in ("fwd", "dgrad", "wgrad"))
    if level == 2:
        assert strats[2] == "BF16"
    p = ah.Params(oe_k=k, level=level)
    xd, wd, gd = dev_bf16(x), dev_bf16(w), dev_bf16(gy)
    outs32 = ah.linear_layer(xd, wd, gd, strats, p, out_dtype=torch.float32)
    outs16 = ah.linear_layer(xd, wd, gd, strats, p, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    for path, s, o32, o16 in zip(("fwd", "dgrad", "wgrad"), strats, outs32, outs16):
        # bf16 output = RN_bf16 of the fp32 accumulator output (same accumulator, epilogue rounding)
        assert torch.equal(o16, o32.to(torch.bfloat16)), (path, s)
        sampled_check(path, s, o32.cpu().numpy(), x, w, gy, k, rng)


def test_linear_layer_graph_replay_bitwise():
    T, d_in, d_out = 2048, 1024, 2048
    x, _ = synth.operand(T, d_in, "C", "X", case_id=601)
    w, _ = synth.operand(d_out, d_in, "N", "W", case_id=602)
    gy, _ = synth.operand(T, d_out, "R", "GY", case_id=603)
    strats = ("IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT")
    p = ah.Params(oe_k=64)
    xd, wd, gd = dev_bf16(x), dev_bf16(w), dev_bf16(gy)
    ws = ah.Workspace(ah.layer_workspace_bytes(T, d_in, d_out, strats, p), DEV)
    eager = ah.linear_layer(xd, wd, gd, strats, p, ws=ws)
    outs = tuple(torch.empty_like(o) for o in eager)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ah.linear_layer(xd, wd, gd, strats, p, out=outs, ws=ws)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ah.linear_layer(xd, wd, gd, strats, p, out=outs, ws=ws)
    for o in outs:
        o.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, outs):
        assert torch.equal(a, b)


@pytest.mark.slow
@pytest.mark.parametrize("rows,cols,pattern", [(16384, 2048, "R"), (16384, 512, "C"), (2048, 8192, "N")])
def test_calibration_full_size(rows, cols, pattern):
    # the calibration pass (a1) at bench sizes: stats tiles, fixed-order partial folds and CV
    # terms against the oracle's fp64 CVs, and the classification
    t, _ = synth.operand(rows, cols, pattern, "GY", case_id=700 + rows // 1024 + cols // 64)
    pat, cvr, cvc = ah.calibrate(dev_bf16(t))
    orow, ocol = O.cv_row_col(t)
    assert abs(cvr - orow) <= 1e-9 * max(1, orow) and abs(cvc - ocol) <= 1e-9 * max(1, ocol)
    assert pat == O.classify(t) == pattern
