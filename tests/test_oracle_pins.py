"""Pins for the CPU oracle (tests/ -m "not gpu").

Each test checks the oracle against something other than itself: a closed form, an
invariant the paper states, a golden fixture with its citation, or brute force on a
tiny input. Chosen so that a dropped term, a wrong sign or index, or a transposed
operand in the oracle fails at least one of them.
"""
import itertools
import math

import numpy as np
import pytest

import oracle as O
import synth
from conftest import golden


# --------------------------------------------------------------------------- Hadamard
def test_hadamard_orthogonality_exact():
    # P:93 "H_k^T H_k = I"; unnormalised Sylvester H satisfies H H^T = n I exactly.
    for b in (2, 4, 8, 16, 32):
        h = O.hadamard_matrix(b, normalized=False)
        assert set(np.unique(h)) == {-1.0, 1.0}
        np.testing.assert_array_equal(h @ h.T, b * np.eye(b))


def test_hadamard_symmetric_involution():
    h = O.hadamard_matrix(32)
    np.testing.assert_array_equal(h, h.T)
    np.testing.assert_allclose(h @ h, np.eye(32), atol=1e-14)


def test_hadamard_h2_example():
    # block size 2, row [1, 1] -> [sqrt2, 0]
    y = O.iht_dense(np.array([[1.0, 1.0]]), b=2)
    np.testing.assert_allclose(y, [[math.sqrt(2.0), 0.0]], atol=1e-15)


def test_fwht_closed_forms():
    e0 = np.zeros((1, 32))
    e0[0, 0] = 1.0
    np.testing.assert_allclose(O.iht_dense(e0), np.full((1, 32), 1 / math.sqrt(32)), atol=1e-15)
    ones = np.ones((1, 32))
    want = np.zeros((1, 32))
    want[0, 0] = math.sqrt(32)
    np.testing.assert_allclose(O.iht_dense(ones), want, atol=1e-13)
    # natural ordering: row j of H is the Walsh function with sign (-1)^popcount(i&j)
    for j in (1, 5, 31):
        ej = np.zeros((1, 32))
        ej[0, j] = 1.0
        signs = np.array([(-1) ** bin(i & j).count("1") for i in range(32)])
        np.testing.assert_allclose(O.iht_dense(ej)[0], signs / math.sqrt(32), atol=1e-15)


def test_fwht_spec_matches_dense_within_bound():
    # fp32 butterflies vs fp64 dense, error <= ~1.05e-7 x block L2 norm
    x, _ = synth.operand(64, 512, "N", "X", case_id=3, bf16=False)
    y32 = O.fwht_fp32_spec(x).astype(np.float64)
    y64 = O.iht_dense(x)
    err = np.abs(y32 - y64).reshape(64, 16, 32).max(-1)
    nrm = np.linalg.norm(x.astype(np.float64).reshape(64, 16, 32), axis=-1)
    assert np.all(err <= 2.0e-7 * nrm + 1e-30)
    assert np.linalg.norm(y32 - y64) / np.linalg.norm(y64) < 1e-6


def test_fwht_spec_involution_and_norm():
    x, _ = synth.operand(8, 256, "C", "X", case_id=4)
    y = O.fwht_fp32_spec(O.fwht_fp32_spec(x))
    np.testing.assert_allclose(y, x, rtol=0, atol=2e-5 * np.abs(x).max())
    np.testing.assert_allclose(np.linalg.norm(O.iht_dense(x)), np.linalg.norm(x.astype(np.float64)), rtol=1e-12)


def test_iht_exact_with_identity_quantiser():
    # A H_k . H_k^T B = A B in infinite precision
    a, _ = synth.operand(48, 256, "C", "X", case_id=5, bf16=False)
    b, _ = synth.operand(40, 256, "N", "W", case_id=6, bf16=False)
    ah = O.iht_dense(a)
    bh = O.iht_dense(b)                      # B_store rows: (H^T B)^T = B^T H
    np.testing.assert_allclose(ah @ bh.T, a.astype(np.float64) @ b.astype(np.float64).T,
                               rtol=1e-12, atol=1e-12)


def test_iht_is_blockwise_not_full():
    # P:761 "block size 32": mixing never crosses a 32-block boundary
    x = np.zeros((1, 128))
    x[0, 40] = 1.0
    y = O.iht_dense(x)
    assert np.all(y[0, :32] == 0) and np.all(y[0, 64:] == 0)
    assert np.all(np.abs(y[0, 32:64]) > 0)


# --------------------------------------------------------------------------- quantiser
def test_e2m1_tie_and_saturation_table():
    for v, mag, code in golden("e2m1_ties.txt"):
        c = O.e2m1_code(np.array([float(v)]))[0]
        assert c == int(code), (v, c)
        assert O.E2M1_VALUES[c & 7] == float(mag)
        cn = O.e2m1_code(np.array([-float(v)]))[0]
        assert cn == (int(code) | 8)


def test_e2m1_nearest_bruteforce_grid():
    # brute force: for every v on a fine grid the chosen value is a nearest codebook value
    v = np.linspace(-9, 9, 14401)
    c = O.e2m1_code(v)
    val = np.where(c & 8, -1.0, 1.0) * O.E2M1_VALUES[c & 7]
    clipped = np.clip(v, -6, 6)
    dist = np.abs(clipped[:, None] - np.concatenate([O.E2M1_VALUES, -O.E2M1_VALUES])[None])
    assert np.all(np.abs(val - clipped) <= dist.min(1) + 1e-15)


def test_e2m1_representable_roundtrip_all_codes():
    for code in range(16):
        mag = O.E2M1_VALUES[code & 7]
        v = -mag if code & 8 else mag
        got = O.e2m1_code(np.array([v]))[0]
        if mag == 0.0:
            assert got & 7 == 0 and (got >> 3) == (code >> 3)   # +0 -> 0x0, -0 -> 0x8
        else:
            assert got == code


def test_scale_rule_ocp_property_all_exponents():
    # OCP MX: e chosen so amax / 2^e lies in [4, 8) (emax of E2M1 = 2), clamped to [-127,127]
    amaxes = []
    for ex in range(-149, 128):
        for m in (1.0, 1.5, 1.9999999):
            v = np.float32(m) * np.float32(2.0) ** ex if ex > -127 else np.float32(np.ldexp(m, ex))
            if np.isfinite(v) and v > 0:
                amaxes.append(float(v))
    amaxes = np.array(amaxes)
    e = O.mx_scale_exponent(amaxes)
    r = amaxes / np.exp2(e.astype(np.float64))
    unclamped = e > -127
    assert np.all((r[unclamped] >= 4) & (r[unclamped] < 8))
    assert np.all(r[~unclamped] < 8)
    assert e.max() <= 127 and e.min() >= -127
    assert O.mx_scale_exponent(np.array([0.0]))[0] == 0


def test_zero_block():
    codes, sc = O.quantize_mxfp4(np.zeros((2, 64)))
    assert np.all(codes == 0) and np.all(sc == 127)


def test_quantiser_properties():
    y, _ = synth.operand(32, 256, "C", "X", case_id=7, bf16=False)
    c1, s1 = O.quantize_mxfp4(y)
    dq = O.dequantize_mxfp4(c1, s1)
    # idempotence
    c2, s2 = O.quantize_mxfp4(dq)
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_array_equal(s1, s2)
    # sign symmetry
    cn, sn = O.quantize_mxfp4(-y)
    np.testing.assert_array_equal(cn, c1 ^ 8)
    np.testing.assert_array_equal(sn, s1)
    # power-of-two equivariance
    for j in (-3, 5):
        cj, sj = O.quantize_mxfp4(y * 2.0 ** j)
        np.testing.assert_array_equal(cj, c1)
        np.testing.assert_array_equal(sj.astype(int), s1.astype(int) + j)
    # error bound under the floor-scale rule: |x - dq| <= 2 * 2^e (saturation region (6,8)*2^e)
    e = s1.astype(np.float64) - 127
    err = np.abs(y.astype(np.float64) - dq).reshape(32, 8, 32).max(-1)
    assert np.all(err <= 2.0 * np.exp2(e))


def test_saturation_example_spec_bound_is_wrong():
    # block amax 7.99 * 2^e -> scale e, value saturates to 6 * 2^e: error ~2 * 2^e (S:136 is wrong)
    y = np.zeros((1, 32))
    y[0, 0] = 7.99
    c, s = O.quantize_mxfp4(y)
    assert s[0, 0] == 127 and c[0, 0] == 7
    assert abs(7.99 - O.dequantize_mxfp4(c, s)[0, 0]) > 1.9


def test_pack_unpack():
    rng = np.random.default_rng(0)
    c = rng.integers(0, 16, size=(4, 64)).astype(np.uint8)
    p = O.pack_codes(c)
    assert p.shape == (4, 32)
    assert p[0, 0] == (c[0, 0] | (c[0, 1] << 4))      # element 2j low nibble
    np.testing.assert_array_equal(O.unpack_codes(p), c)


def test_round_bf16_known_values():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 2 ** -7, 1.0 + 3 * 2 ** -8, -2.5, 3.0e38], dtype=np.float32)
    want = np.array([1.0, 1.0, 1.0 + 2 ** -7, 1.0 + 2 ** -6, -2.5, 2.9975006e38])
    got = O.round_bf16(x)
    np.testing.assert_allclose(got[:5], want[:5], rtol=0, atol=0)
    assert abs(got[5] / 3.0e38 - 1) < 2 ** -8


# --------------------------------------------------------------------------- FOID / OE
def test_foid_single_outlier_row_first_and_clamp():
    x, pl = synth.operand(64, 128, "R", "X", case_id=8, count=1)
    idx = O.foid_indices(x, k=1)
    np.testing.assert_array_equal(idx, pl.rows)
    np.testing.assert_array_equal(O.foid_indices(x, k=1000), np.arange(64))
    assert len(O.foid_indices(x, k=0)) == 0


def test_foid_planted_rows_always_selected():
    for case in range(5):
        x, pl = synth.operand(2048, 256, "R", "X", case_id=100 + case, count=5)
        idx = O.foid_indices(x, k=8)
        assert set(pl.rows) <= set(idx) and len(idx) == 8
        assert np.all(np.diff(idx) > 0)


def test_foid_bruteforce_and_ties():
    # tiny brute force: keys from the textbook population variance of the first p entries
    rng = np.random.default_rng(1)
    x = rng.standard_normal((12, 80)).astype(np.float32)
    x[3] = x[7]                      # exact tie -> lower index wins
    keys = [float(np.var(x[i, :64].astype(np.float64))) for i in range(12)]
    np.testing.assert_allclose(O.foid_keys(x), keys, rtol=1e-13)
    for k in range(13):
        got = O.foid_indices(x, k=k)
        ranked = sorted(range(12), key=lambda i: (-keys[i], i))[:k]
        assert list(got) == sorted(ranked)
    # only the probe prefix matters ("first 64 elements")
    y = x.copy()
    y[:, 64:] *= 1000
    np.testing.assert_array_equal(O.foid_indices(y, 4), O.foid_indices(x, 4))
    # short rows: probe clamps to K
    np.testing.assert_allclose(O.foid_keys(x[:, :32]), np.var(x[:, :32].astype(np.float64), axis=1), rtol=1e-13)


def test_oe_split_partition_exact():
    x, _ = synth.operand(32, 64, "R", "X", case_id=9)
    idx = O.foid_indices(x, k=4)
    res, out = O.oe_split(x, idx)
    recon = res.copy()
    recon[idx] += out
    np.testing.assert_array_equal(recon.view(np.uint32), x.view(np.uint32))
    assert np.all(res[idx] == 0) and not np.any(np.signbit(res[idx]))


# --------------------------------------------------------------------------- strategy / calibration
def test_strategy_table_golden():
    rows = golden("strategy_table.txt")
    assert len(rows) == 18
    for left, right, level, strat in rows:
        assert O.strategy_for_pair(left, right, int(level)) == strat


def test_cv_closed_forms():
    # constant matrix -> CV 0 -> None; iid Gaussian -> CV = sqrt(pi/2)
    assert O.classify(np.full((64, 64), 3.0)) == "N"
    g = np.random.Generator(np.random.Philox(7)).standard_normal((2048, 2048))
    cr, cc = O.cv_row_col(g)
    assert abs(cr - math.sqrt(math.pi / 2)) < 0.01 and abs(cc - math.sqrt(math.pi / 2)) < 0.01
    assert O.classify(g) == "N"


def test_classify_planted_patterns_and_duality():
    for rows, cols in ((256, 256), (2048, 512), (512, 4096)):
        for p in "RCN":
            t, _ = synth.operand(rows, cols, p, "GY", case_id=11)
            assert O.classify(t) == p
            assert O.classify(t.T) == O.transpose_pattern(p)
            assert O.classify(t * 37.0) == p                      # scale invariance S:261


def test_classify_both_above_tau_closed_forms():
    # The both-above-tau branch of App. A's rule (reading R7: larger CV wins, exact
    # tie -> Row), pinned on 0/1 matrices whose CVs have closed forms. A row (or
    # column) of length n with r ones has mean r/n and population std sqrt(r/n (1 - r/n)), so
    # std / mean|x| = sqrt(n/r - 1) (eps = 1e-8 moves it by < 1e-5). All sums are exact dyadic
    # fractions, so the tie below is exact in fp64 (the tolerances cover eps).
    s3, s7, s15 = math.sqrt(3), math.sqrt(7), math.sqrt(15)
    # identity: every row and column has one 1 of 16 -> CV_row = CV_col = sqrt(15) > tau: tie -> R
    ident = np.eye(16)
    cr, cc = O.cv_row_col(ident)
    assert cr == cc and abs(cr - s15) < 1e-5
    assert O.classify(ident) == "R"
    # identity + row 0 also holding ones at columns 1..3: row 0 has r = 4 (sqrt 3), rows 1..15
    # r = 1 (sqrt 15); columns 1..3 have r = 2 (sqrt 7), the other 13 r = 1 (sqrt 15)
    t = np.eye(16)
    t[0, 1:4] = 1.0
    cr, cc = O.cv_row_col(t)
    want_r, want_c = (s3 + 15 * s15) / 16, (13 * s15 + 3 * s7) / 16     # 3.7392, 3.6429
    assert abs(cr - want_r) < 1e-5 and abs(cc - want_c) < 1e-5
    assert cr > cc > O.TAU
    assert O.classify(t) == "C"          # both above tau, CV_row larger -> Column-wise
    assert O.classify(t.T) == "R"        # transposed: CV_col larger -> Row-wise
    # only one direction above tau: 16 x 4 with a single 1 per row (rows: sqrt(3) < tau;
    # columns: 4 ones of 16 -> sqrt(3) too) -> None; 4 x 64 diagonal-ish: rows sqrt(63) -> C
    assert O.classify(np.tile(np.eye(4), (4, 1))) == "N"
    wide = np.zeros((4, 64))
    wide[np.arange(4), np.arange(4) * 16] = 1.0
    cr, cc = O.cv_row_col(wide)
    assert abs(cr - math.sqrt(63)) < 1e-5 and abs(cc - math.sqrt(3) * 4 / 64) < 1e-5
    assert O.classify(wide) == "C"


def test_majority_vote_examples():
    # SPEC S:257-259
    assert O.majority_vote(["R"] * 30) == "R"
    assert O.majority_vote(["R"] * 16 + ["N"] * 14) == "R"
    assert O.majority_vote(["R"] * 15 + ["C"] * 15) == "R"
    assert O.majority_vote(["N"] * 10 + ["C"] * 10) == "C"
    with pytest.raises(ValueError):
        O.majority_vote([])


def test_table1_census_pins_orientation():
    # tab:pattern_distribution Llama3.2-1B: 112 linears; the per-tensor census
    # (W = N everywhere) of SURVEY §8d config 5 must reproduce the three path columns exactly.
    census = [("N", "C")] * 15 + [("C", "C")] * 69 + [("C", "N")] * 20 + [("C", "R")] * 8
    counts = {p: {} for p in ("fwd", "wgrad", "dgrad")}
    for px, pg in census:
        for path in counts:
            a, b = O.fed_patterns(path, px, "N", pg)
            counts[path][a + b] = counts[path].get(a + b, 0) + 1
    for pair, model, fwd, wgrad, dgrad in golden("table1_census.txt"):
        if model != "llama32_1b":
            continue
        assert counts["fwd"].get(pair, 0) == int(fwd), pair
        assert counts["wgrad"].get(pair, 0) == int(wgrad), pair
        assert counts["dgrad"].get(pair, 0) == int(dgrad), pair


def test_table1_cross_path_identity_all_models():
    # For every model: dgrad-A (G_Y) counts equal swapped wgrad-A (G_Y^T) counts, and
    # fwd-A (X) counts equal wgrad-B (X) counts, as the fed-orientation reading requires.
    t = O.transpose_pattern
    for model in ("llama32_1b", "instella_3b", "llama31_8b"):
        rows = [r for r in golden("table1_census.txt") if r[1] == model]
        fa, wa, wb, da = {}, {}, {}, {}
        for pair, _, fwd, wgrad, dgrad in rows:
            fa[pair[0]] = fa.get(pair[0], 0) + int(fwd)
            wa[pair[0]] = wa.get(pair[0], 0) + int(wgrad)
            wb[pair[1]] = wb.get(pair[1], 0) + int(wgrad)
            da[pair[0]] = da.get(pair[0], 0) + int(dgrad)
        for p in "RCN":
            assert da.get(p, 0) == wa.get(t(p), 0), (model, p)
            assert fa.get(p, 0) == wb.get(p, 0), (model, p)


# --------------------------------------------------------------------------- end-to-end oracle
def _bruteforce_matmul(qa, qb):
    ca, sa = qa
    cb, sb = qb
    m, k = ca.shape
    n = cb.shape[0]
    out = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            s = 0.0
            for t in range(k):
                va = O.E2M1_VALUES[ca[i, t] & 7] * (-1 if ca[i, t] & 8 else 1) * 2.0 ** (int(sa[i, t // 32]) - 127)
                vb = O.E2M1_VALUES[cb[j, t] & 7] * (-1 if cb[j, t] & 8 else 1) * 2.0 ** (int(sb[j, t // 32]) - 127)
                s += va * vb
            out[i, j] = s
    return out


def test_main_product_bruteforce_tiny():
    a, _ = synth.operand(6, 64, "C", "X", case_id=12)
    b, _ = synth.operand(5, 64, "N", "W", case_id=13)
    c, parts = O.adahop_matmul(a, b, O.IHT, return_parts=True)
    np.testing.assert_allclose(c, _bruteforce_matmul(parts["qa"], parts["qb"]), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("strategy", [O.OE_LEFT, O.OE_RIGHT])
def test_oe_disjoint_support_and_scatter(strategy):
    a, _ = synth.operand(128, 256, "R", "X", case_id=14, count=3)
    b, _ = synth.operand(96, 256, "R", "W", case_id=15, count=2)   # B_store rows = columns of B
    c, parts = O.adahop_matmul(a, b, strategy, k=8, return_parts=True)
    idx = parts["idx"]
    if strategy == O.OE_LEFT:
        assert np.all(parts["c_main"][idx, :] == 0)
        np.testing.assert_array_equal(c[idx, :], parts["c_out"])
        # brute-force outlier rows: bf16 dot products
        for t, i in enumerate(idx):
            np.testing.assert_allclose(parts["c_out"][t], b.astype(np.float64) @ a[i].astype(np.float64), rtol=1e-12)
    else:
        assert np.all(parts["c_main"][:, idx] == 0)
        np.testing.assert_array_equal(c[:, idx], parts["c_out"])


def test_oe_full_extraction_is_exact_bf16():
    # k >= dim -> whole product in BF16
    a, _ = synth.operand(16, 64, "N", "X", case_id=16)
    b, _ = synth.operand(24, 64, "N", "W", case_id=17)
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    np.testing.assert_allclose(O.adahop_matmul(a, b, O.OE_LEFT, k=16), exact, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.adahop_matmul(a, b, O.OE_RIGHT, k=24), exact, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.adahop_matmul(a, b, O.BF16), exact, rtol=1e-12, atol=1e-14)


def test_zero_operand_gives_zero():
    a = np.zeros((8, 64), np.float32)
    b, _ = synth.operand(8, 64, "N", "W", case_id=18)
    for s in (O.IHT, O.OE_LEFT, O.OE_RIGHT, O.BF16):
        assert np.all(O.adahop_matmul(a, b, s, k=2) == 0)


def test_oe_reduces_error_on_rn_and_rc():
    # Directional check of Thm OE: with planted row outliers in A, OE-Left
    # beats plain IHT; with column outliers in B (RC pair), OE-Right beats IHT.
    a, _ = synth.operand(256, 256, "R", "X", case_id=19, count=2)
    b, _ = synth.operand(256, 256, "N", "W", case_id=20)
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    e_iht = np.linalg.norm(O.adahop_matmul(a, b, O.IHT) - exact)
    e_oel = np.linalg.norm(O.adahop_matmul(a, b, O.OE_LEFT, k=8) - exact)
    assert e_oel < 0.5 * e_iht
    bc, _ = synth.operand(256, 256, "R", "W", case_id=21, count=2)   # B_store rows = B columns -> C pattern of B
    exact = a.astype(np.float64) @ bc.astype(np.float64).T
    e_iht = np.linalg.norm(O.adahop_matmul(a, bc, O.IHT) - exact)
    e_oer = np.linalg.norm(O.adahop_matmul(a, bc, O.OE_RIGHT, k=8) - exact)
    assert e_oer < e_iht


def test_paths_match_paper_equations():
    # P:75-77 with the identity quantiser replaced by the BF16 strategy: the stored-operand
    # mapping must give Y = X W^T, G_W = G_Y^T X, G_X = G_Y W.
    x, _ = synth.operand(64, 96, "N", "X", case_id=22)
    w, _ = synth.operand(32, 96, "N", "W", case_id=23)
    gy, _ = synth.operand(64, 32, "N", "GY", case_id=24)
    xd, wd, gd = (v.astype(np.float64) for v in (x, w, gy))
    np.testing.assert_allclose(O.linear("fwd", O.BF16, x=x, w=w), xd @ wd.T, rtol=1e-12)
    np.testing.assert_allclose(O.linear("dgrad", O.BF16, w=w, gy=gy), gd @ wd, rtol=1e-12)
    np.testing.assert_allclose(O.linear("wgrad", O.BF16, x=x, gy=gy), gd.T @ xd, rtol=1e-12)


def test_sampled_entries_match_full():
    a, _ = synth.operand(96, 256, "R", "X", case_id=25, count=2)
    b, _ = synth.operand(80, 256, "R", "W", case_id=26, count=2)
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 96, 200)
    cols = rng.integers(0, 80, 200)
    for s in (O.IHT, O.OE_LEFT, O.OE_RIGHT, O.BF16):
        full = O.adahop_matmul(a, b, s, k=4)
        np.testing.assert_allclose(O.sampled_entries(a, b, s, rows, cols, k=4), full[rows, cols],
                                   rtol=1e-12, atol=1e-300)


def test_gamma_definition():
    a = np.ones((4, 4))
    assert O.gamma(a) == 1.0
    a[0, 0] = 4.0
    assert abs(O.gamma(a) - 16 * 16 / (15 + 16)) < 1e-12


# ---------------------------------------------------------------------- outlier counts / adaptive k [R16]
def test_outlier_counts_closed_forms():
    # planted channels (x100, the synth recipe) are exactly the counted ones in the pattern's
    # direction at Llama shapes; Gaussian bulk rows / columns (max ~ 4 sigma against 32 x mean|x|
    # ~ 25 sigma) are never counted. (Across the pattern, App. D's definition flags most
    # channels: every column of a Row-pattern tensor holds an outlier-row entry.)
    for rows, cols in ((2048, 512), (4096, 2048), (512, 4096)):
        for pat in "RCN":
            t, planted = synth.operand(rows, cols, pat, "X", case_id=1300 + rows % 7)
            r, c = O.outlier_counts(t)
            if pat == "R":
                assert r == len(planted.rows), (rows, cols, r)
            elif pat == "C":
                assert c == len(planted.cols), (rows, cols, c)
            else:
                assert (r, c) == (0, 0)
    # transpose swaps the counts; a positive scale leaves them unchanged
    t, _ = synth.operand(1024, 768, "R", "GY", case_id=1310)
    assert O.outlier_counts(t.T) == tuple(reversed(O.outlier_counts(t)))
    assert O.outlier_counts(t * 2.0 ** 37) == O.outlier_counts(t)
    # a single entry: one row and one column; a constant matrix: none
    z = np.zeros((64, 64))
    z[5, 9] = 1.0
    assert O.outlier_counts(z) == (1, 1)
    assert O.outlier_counts(np.ones((64, 64))) == (0, 0)


def test_adaptive_k_rounding_and_clamps():
    assert [O.adaptive_k(c) for c in (0, 1, 15, 16, 17, 33, 48, 49, 64, 65, 1000)] == \
        [16, 16, 16, 16, 32, 48, 48, 64, 64, 64, 64]
    assert O.adaptive_k(5, k_max=256) == 16 and O.adaptive_k(200, k_max=256) == 208
