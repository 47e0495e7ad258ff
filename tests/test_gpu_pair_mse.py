"""Nine-pair error sweep on the GPU path (P:161-163 Imp metric), see
tests/pair_mse_sweep.py. Pins: (1) the GPU IHT error equals the oracle's (the codes are bit-exact;
only the fp32 vs fp64 accumulation differs); (2) Thm. OE: extracting the
outer-dimension outliers beats IHT alone — OE-Left for row-outlier A (RR, RC, RN), OE-Right
for column-outlier B (RC, CC, NC); (3) Prop. transform effectiveness: IHT along K
lowers the error when the outliers lie along K on one side only (CN, NR)."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pair_mse_sweep as pair_mse  # noqa: E402


@pytest.fixture(scope="module")
def table():
    return {r["pair"]: r for r in pair_mse.sweep(seeds=2)}


def test_gpu_iht_error_equals_oracle(table):
    for pair, r in table.items():
        assert abs(r["iht_gpu_vs_oracle"] - 1.0) <= 1e-3, pair


@pytest.mark.parametrize("pair,strategy", [("RR", "OE_LEFT_IHT"), ("RC", "OE_LEFT_IHT"), ("RN", "OE_LEFT_IHT"),
                                           ("RC", "OE_RIGHT_IHT"), ("CC", "OE_RIGHT_IHT"), ("NC", "OE_RIGHT_IHT")])
def test_oe_beats_iht_on_outer_outliers(table, pair, strategy):
    r = table[pair]
    assert r[f"relmse_{strategy}"] < 0.5 * r["relmse_IHT"], (pair, strategy)


@pytest.mark.parametrize("pair", ["CN", "NR"])
def test_iht_improves_inner_outliers(table, pair):
    assert table[pair]["imp_iht_pct"] > 10.0, pair
