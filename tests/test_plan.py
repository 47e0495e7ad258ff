"""CPU tests of the calibration plan's host logic (§5.1): the library's vote and
fed-orientation / strategy mapping, driven by per-step pattern records, must reproduce the
Llama-3.2-1B census of Table 1 (tests/golden/table1_census.txt) from the config-5
per-tensor patterns, also when some calibration steps disagree; and the plan persists."""
import random

import pytest

import oracle as O
import synth
from conftest import golden

ah = pytest.importorskip("paper_2604_02525_b200")
plan_mod = pytest.importorskip("paper_2604_02525_b200.plan")


def test_layer_strategies_match_oracle_orientation_and_table():
    for px in "RCN":
        for pw in "RCN":
            for pg in "RCN":
                for level in (1, 2):
                    strats, fed = ah.layer_strategies(px, pw, pg, level)
                    for path, s, pair in zip(("fwd", "dgrad", "wgrad"), strats, fed):
                        a, b = O.fed_patterns(path, px, pw, pg)
                        assert pair == a + b
                        assert s == O.strategy_for_pair(a, b, level)
    with pytest.raises(ValueError):
        ah.layer_strategies("R", "N", "N", 3)


def _census_records(noise_steps=0, steps=30, seed=0):
    rnd = random.Random(seed)
    linears, rec = [], {}
    for layer, name, px, pw, pg in synth.llama32_1b_census_patterns():
        key = f"l{layer}.{name}"
        d_in, d_out = next((a, b) for n, a, b in synth.LLAMA32_1B["linears"] if n == name)
        linears.append((key, d_in, d_out))
        for t, p in zip(plan_mod.TENSORS, (px, pw, pg)):
            r = [p] * steps
            for i in rnd.sample(range(steps), noise_steps):   # steps where the detector disagreed
                r[i] = rnd.choice([q for q in "RCN" if q != p])
            rec[(key, t)] = r
    return linears, rec


@pytest.mark.parametrize("noise", [0, 9])
def test_plan_reproduces_table1_census(noise):
    linears, rec = _census_records(noise_steps=noise)
    plan = plan_mod.plan_from_patterns(linears, rec, level=1)
    census = plan.census()
    want = {p: {} for p in ("fwd", "wgrad", "dgrad")}
    for pair, model, fwd, wgrad, dgrad in golden("table1_census.txt"):
        if model == "llama32_1b":
            for path, v in (("fwd", fwd), ("wgrad", wgrad), ("dgrad", dgrad)):
                if int(v):
                    want[path][pair] = int(v)
    for path in want:
        assert census[path] == want[path], path
    # strategy counts follow tab:strategy_summary: wgrad RN -> OE-L, RC / CC -> OE-R, NC -> OE-R
    n_oe_r = sum(1 for lp in plan.linears if lp.strategies[2] == "OE_RIGHT_IHT")
    assert n_oe_r == 69 + 20 + 8


def test_plan_json_round_trip(tmp_path):
    linears, rec = _census_records(noise_steps=3)
    plan = plan_mod.plan_from_patterns(linears, rec, level=2)
    f = tmp_path / "plan.json"
    plan.save(str(f))
    back = plan_mod.Plan.load(str(f))
    assert back.census() == plan.census() and back.level == 2 and back.steps == 30
    assert [lp.strategies for lp in back.linears] == [lp.strategies for lp in plan.linears]
    # Lv2: the 8 CC wgrads run in BF16
    assert sum(1 for lp in back.linears if lp.strategies[2] == "BF16") == 8


def test_adaptive_k_matches_oracle_and_picks_the_oe_operand():
    # plan.adaptive_k is the host copy of oracle.adaptive_k (DESIGN R16)
    for c in (0, 1, 15, 16, 17, 40, 63, 64, 65, 500):
        assert plan_mod.adaptive_k(c) == O.adaptive_k(c)
    out = {"X": [3, 40], "W": [0, 17], "G_Y": [5, 70]}
    # wgrad OE-Right sizes k from X's columns; dgrad OE-Left from G_Y's rows; the largest wins
    assert plan_mod.layer_oe_k(("IHT", "IHT", "OE_RIGHT_IHT"), out) == 48
    assert plan_mod.layer_oe_k(("IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT"), out) == 48
    assert plan_mod.layer_oe_k(("IHT", "OE_LEFT_IHT", "IHT"), out) == 16
    assert plan_mod.layer_oe_k(("IHT", "IHT", "OE_LEFT_IHT"), out) == 64   # G_Y's columns (70) -> clamp
    assert plan_mod.layer_oe_k(("IHT", "OE_RIGHT_IHT", "BF16"), out) == 32  # W's columns (17)
    assert plan_mod.layer_oe_k(("IHT", "IHT", "IHT"), out) == 0
