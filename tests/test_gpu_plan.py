"""Config 5 calibration on the GPU (§5.1): 30 calibration steps over the 16 x 7 linears of
Llama-3.2-1B (fresh noise every step, outlier channels fixed per tensor, a few steps without any
planted outliers), each tensor classified by adahop_calibrate on the device, voted and mapped to
strategies by the library — the recovered census must be Table 1's."""
import pytest

import synth
from conftest import golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_02525_b200 as ah  # noqa: E402
from paper_2604_02525_b200 import plan as plan_mod  # noqa: E402

DEV = torch.device("cuda:0")


def test_calibration_plan_recovers_table1_census():
    T, steps = 1024, 30
    quiet = {3, 11, 19, 27}           # steps whose batch carries no outliers (the detector says N)
    cfg = synth.llama32_1b_census_patterns()
    dims = {n: (a, b) for n, a, b in synth.LLAMA32_1B["linears"]}
    linears = [(f"l{layer}.{name}", *dims[name]) for layer, name, *_ in cfg]
    cal = plan_mod.Calibrator(linears, steps=steps, params=ah.Params(), device=DEV)
    ws = {}
    for i, (layer, name, px, pw, pg) in enumerate(cfg):
        d_in, d_out = dims[name]
        key = f"l{layer}.{name}"
        w = synth.operand_torch(d_out, d_in, pw, "W", 20000 + i, DEV)
        x = ws.setdefault(("x", d_in), torch.empty((T, d_in), dtype=torch.bfloat16, device=DEV))
        gy = ws.setdefault(("gy", d_out), torch.empty((T, d_out), dtype=torch.bfloat16, device=DEV))
        for s in range(steps):
            synth.operand_torch(T, d_in, "N" if s in quiet else px, "X", 100000 * s + i, DEV, plant_seed=30000 + i, out=x)
            synth.operand_torch(T, d_out, "N" if s in quiet else pg, "GY", 100000 * s + 50000 + i, DEV,
                                plant_seed=40000 + i, out=gy)
            cal.record(s, key, x, w, gy)
    plan = cal.plan(level=1)
    census = plan.census()
    want = {p: {} for p in ("fwd", "wgrad", "dgrad")}
    for pair, model, fwd, wgrad, dgrad in golden("table1_census.txt"):
        if model == "llama32_1b":
            for path, v in (("fwd", fwd), ("wgrad", wgrad), ("dgrad", dgrad)):
                if int(v):
                    want[path][pair] = int(v)
    assert census == {p: want[p] for p in census}
    # every tensor's vote: 26 planted steps agree, the 4 quiet ones say N
    for lp, (_, _, px, pw, pg) in zip(plan.linears, cfg):
        assert lp.patterns == {"X": px, "W": pw, "G_Y": pg}
        for t, p in zip(("X", "G_Y"), (px, pg)):
            if p != "N":
                assert lp.votes[t] == {p: 26, "N": 4}
    # adaptive k (DESIGN R16): T = 1024 tokens plant 2 channels per C tensor (0.1 % of 2048 / 8192
    # columns: 3 / 9) and 2 rows per R tensor -> every OE operand's count rounds up to k = 16
    for lp in plan.linears:
        assert lp.oe_k == (16 if any(s.startswith("OE") for s in lp.strategies) else 0), (lp.name, lp.strategies)


def test_outlier_counts_match_oracle():
    # adahop_calibrate_batch_outliers against oracle.outlier_counts on planted tensors (the counts in
    # the pattern's direction are the planted channels; across it App. D flags most channels)
    import numpy as np
    import oracle as O
    shapes = [(2048, 512, "R"), (4096, 2048, "C"), (512, 4096, "R"), (1024, 768, "N"), (16384, 512, "C")]
    host, ts = [], []
    for i, (r, c, p) in enumerate(shapes):
        a, _ = synth.operand(r, c, p, "GY", case_id=1400 + i)
        host.append(a)
        ts.append(torch.from_numpy(a).to(DEV, torch.bfloat16))
    ws = torch.empty(ah.calibrate_batch_workspace_bytes([t.shape for t in ts]), dtype=torch.uint8, device=DEV)
    cv = torch.empty((len(ts), 4), dtype=torch.float64, device=DEV)
    pat = torch.empty(len(ts), dtype=torch.uint8, device=DEV)
    cnt = torch.empty((len(ts), 2), dtype=torch.int32, device=DEV)
    ah.calibrate_batch_async(ts, ws, cv, pat)
    ah.calibrate_batch_outliers_async([t.shape for t in ts], ws, cnt)
    got = cnt.cpu().tolist()
    for (r, c, p), a, g in zip(shapes, host, got):
        want = O.outlier_counts(np.asarray(a, np.float64))   # the bf16 values the GPU saw
        assert tuple(g) == want, (r, c, p, g, want)
