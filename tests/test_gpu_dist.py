"""Multi-rank GPU parity of the data-parallel path: two gloo ranks share cuda:0
and run the CUDA library on their token shards.

* wgrad: the all-reduced G_W equals the sum over shards of the oracle's per-shard AdaHOP wgrad
  (rank-local FOID and Hadamard blocks; eq:backward_gw P:76), within the north star's 1e-3
  relative Frobenius error for fp32 partials; bf16 partials (rounded once per rank, summed in
  bf16) stay within a measured 5e-3.
* layer call: every rank's Y / G_X equal the oracle on its own shard; G_W as above.
* calibration: stats -> all-reduce -> classify -> all-reduce -> classify_sums (all arithmetic in
  the library) gives the oracle's pattern and CVs of the WHOLE tensor on every rank.
"""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from _mp import spawn  # noqa: E402

T, D_IN, D_OUT, K_OE = 1024, 384, 256, 16
TOL_OUT = 1e-3


def _rel(got, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(np.asarray(got, np.float64) - ref) / np.linalg.norm(ref))


def _inputs():
    x, _ = synth.operand(T, D_IN, "C", "X", case_id=911)
    w, _ = synth.operand(D_OUT, D_IN, "N", "W", case_id=912)
    gy, _ = synth.operand(T, D_OUT, "C", "GY", case_id=913)
    return x, w, gy


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0", torch.bfloat16)


def _dp_wgrad(rank, world):
    import paper_2604_02525_b200 as ah
    import paper_2604_02525_b200.dist as ahd
    torch.cuda.set_device(0)
    x, w, gy = _inputs()
    t0, t1 = ahd.token_shard(T, world, rank)
    p = ah.Params(oe_k=K_OE)
    out = {}
    for dt in (torch.float32, torch.bfloat16):
        lin = ahd.DataParallelLinear({"fwd": "IHT", "dgrad": "IHT", "wgrad": "OE_RIGHT_IHT"}, params=p)
        gw = lin.wgrad(_dev(gy[t0:t1]), _dev(x[t0:t1]), out_dtype=dt)
        torch.cuda.synchronize()
        out[str(dt)] = gw.float().cpu().numpy()
    # the layer call on the shard (fwd / dgrad local, wgrad partial all-reduced)
    strats = ("IHT", "IHT", "OE_RIGHT_IHT")
    y, gx, gwl = ah.linear_layer(_dev(x[t0:t1]), _dev(w), _dev(gy[t0:t1]), strats, p, out_dtype=torch.float32)
    ahd.allreduce_wgrad(gwl)
    torch.cuda.synchronize()
    out["layer"] = (y.cpu().numpy(), gx.cpu().numpy(), gwl.cpu().numpy())
    return out


def test_wgrad_allreduce_equals_sum_of_shard_oracles_on_gpu():
    out = spawn(_dp_wgrad)
    x, w, gy = _inputs()
    shards = [(a, b) for a, b in (__import__("paper_2604_02525_b200.dist", fromlist=["x"]).token_shard(T, 2, r)
                                  for r in range(2))]
    want = sum(O.linear("wgrad", O.OE_RIGHT, x=x[a:b], gy=gy[a:b], k=K_OE) for a, b in shards)
    for r in (0, 1):
        assert _rel(out[r][str(torch.float32)], want) <= TOL_OUT
        assert _rel(out[r][str(torch.bfloat16)], want) <= 5e-3
        y, gx, gwl = out[r]["layer"]
        a, b = shards[r]
        assert _rel(y, O.linear("fwd", O.IHT, x=x[a:b], w=w, k=K_OE)) <= TOL_OUT
        assert _rel(gx, O.linear("dgrad", O.IHT, w=w, gy=gy[a:b], k=K_OE)) <= TOL_OUT
        assert _rel(gwl, want) <= TOL_OUT
    # every rank holds the same reduced gradient
    np.testing.assert_array_equal(out[0][str(torch.float32)], out[1][str(torch.float32)])
    np.testing.assert_array_equal(out[0]["layer"][2], out[1]["layer"][2])


def _dp_calib(rank, world):
    import paper_2604_02525_b200.dist as ahd
    torch.cuda.set_device(0)
    res = {}
    for i, p in enumerate("RCN"):
        t, _ = synth.operand(2048, 512, p, "GY", case_id=920 + i)
        a, b = ahd.token_shard(2048, world, rank)
        step = ahd.calibrate_sharded(_dev(t[a:b]), 2048)
        res[p] = (step.pattern, step.cv_row, step.cv_col)
    return res


def test_sharded_calibration_on_gpu_matches_whole_tensor_oracle():
    out = spawn(_dp_calib)
    for i, p in enumerate("RCN"):
        t, _ = synth.operand(2048, 512, p, "GY", case_id=920 + i)
        cr, cc = O.cv_row_col(t)
        for r in (0, 1):
            pat, cvr, cvc = out[r][p]
            assert pat == O.classify(t) == p
            assert abs(cvr - cr) <= 1e-9 * cr and abs(cvc - cc) <= 1e-9 * cc
