"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs. Bit-exact for codes / scales / index sets; 1e-6 relative for the Hadamard
output; 1e-3 relative Frobenius for linear outputs (north star), on fp32 outputs
(a bf16 output alone carries ~1.7e-3 rounding).
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
TOL_OUT = 1e-3      # north star: linear outputs within 1e-3 relative Frobenius
TOL_HAD = 1e-6      # north star: Hadamard outputs within 1e-6 relative


def dev_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, torch.bfloat16)


def dev_f32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(DEV)


def rel_fro(got, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(np.asarray(got, np.float64) - ref) / max(np.linalg.norm(ref), 1e-300))


# ======================================================================= E2M1 conversion
def test_e2m1_hw_conversion_matches_oracle_rule():
    ties = [0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0, 7.0, 7.99, 8.0, 1e30, 0.0]
    grid = np.linspace(-9, 9, 180001)
    rnd = np.random.default_rng(0).standard_normal(1 << 20) * 3
    v = np.concatenate([ties, -np.array(ties), grid, rnd, np.nextafter(np.array(ties), 10),
                        np.nextafter(np.array(ties), -10)]).astype(np.float32)
    hw, sw = ah.debug_e2m1(dev_f32(v))
    want = O.e2m1_code(v.astype(np.float64))
    np.testing.assert_array_equal(sw.cpu().numpy(), want)
    np.testing.assert_array_equal(hw.cpu().numpy(), want)


def test_e2m1_hw_vs_rule_exhaustive_fp32():
    # every finite fp32 bit pattern: hardware cvt == the stated rounding rule
    mism, first = ah.debug_e2m1_exhaustive(0, 1 << 32)
    assert mism == 0, f"{mism} mismatches, first at bits 0x{first:08x}"


# ======================================================================= IHT + quant
def _quant_case(R, K, dtype, k_strided, pattern="C", case=0, zero_rows=None):
    x, _ = synth.operand(R, K, pattern, "X", case_id=case, bf16=(dtype == "bf16"))
    xin = x.T.copy() if k_strided else x
    t = dev_bf16(xin) if dtype == "bf16" else dev_f32(xin)
    codes, scales, had = ah.debug_iht_quant(t, k_strided=k_strided, zero_rows=zero_rows, want_had=True)
    torch.cuda.synchronize()
    xs = x.copy()
    if zero_rows is not None and len(zero_rows):
        xs[np.asarray(zero_rows)] = 0.0
    return xs, codes.cpu().numpy(), scales.cpu().numpy(), had.cpu().numpy()


@pytest.mark.parametrize("k_strided", [False, True])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("R,K", [(300, 1024), (77, 96), (128, 256), (1031, 2080)])
def test_iht_quant_bitexact(R, K, dtype, k_strided):
    xs, codes, scales, had = _quant_case(R, K, dtype, k_strided, case=R + K)
    if dtype == "f32":
        # (b) butterfly kernels: the fp32 Hadamard output equals the oracle's fp32 butterfly
        # spec bitwise. (bf16 sources take the tensor-core kernel, whose fp32 accumulation
        # order is the hardware's: protocol (a) only, R2.)
        np.testing.assert_array_equal(had.view(np.uint32), O.fwht_fp32_spec(xs).view(np.uint32))
    # Hadamard within 1e-6 relative of the fp64 dense transform
    assert rel_fro(had, O.iht_dense(xs)) <= TOL_HAD
    # (a) codes and E8M0 scales bit-exact given the same fp32 input
    oc, osc = O.quantize_mxfp4(had)
    np.testing.assert_array_equal(scales, osc)
    np.testing.assert_array_equal(codes, O.pack_codes(oc))


@pytest.mark.parametrize("k_strided", [False, True])
def test_iht_quant_residual_mask(k_strided):
    zr = [0, 5, 6, 129, 299]
    xs, codes, scales, had = _quant_case(300, 512, "bf16", k_strided, pattern="R", case=7, zero_rows=zr)
    assert rel_fro(had, O.iht_dense(xs)) <= TOL_HAD
    oc, osc = O.quantize_mxfp4(had)
    np.testing.assert_array_equal(codes, O.pack_codes(oc))
    np.testing.assert_array_equal(scales, osc)
    assert np.all(codes[zr] == 0) and np.all(scales[zr] == 127)   # +0 codes, e = 0


@pytest.mark.parametrize("R,C,masks", [(256, 512, False), (384, 160, True), (2048, 1024, True),
                                        (4096, 96, True), (256, 384, "dense"), (544, 2048, "wide"),
                                        (96, 1056, "wide")])
def test_quant_dual_equals_single_orientation(R, C, masks):
    # one pass over T emitting both layouts == the row quantisation of T and of T^T, bitwise,
    # and both == the oracle quantiser on the Hadamard output (protocol (a)); "dense" puts more
    # extracted rows + columns in one tile than the kernel's slice staging ring holds; "wide"
    # (>= C / 128 extracted columns: a slice over most of every row's lines, ragged 256-column chunks)
    x, _ = synth.operand(R, C, "R", "X", case_id=R * 7 + C, bf16=True)
    if masks == "wide":
        g = np.random.default_rng(R + C)
        rz, cz = sorted({0, R // 3, R - 1}), sorted(g.choice(C, size=max(C // 32, 9), replace=False).tolist())
    elif masks == "dense":
        rz, cz = list(range(0, R, 2)), list(range(0, C, 3))
    else:
        rz = sorted({0, 3, R // 2, R - 1}) if masks else None
        cz = sorted({1, C // 3, C - 2}) if masks else None
    t = dev_bf16(x)
    qr, sr, qc, sc, slr, slc = ah.debug_quant_dual(t, row_zero=rz, col_zero=cz, want_slices=True)
    codes_r, scales_r, had_r = ah.debug_iht_quant(t, zero_rows=rz, want_had=True)
    codes_c, scales_c, had_c = ah.debug_iht_quant(t, k_strided=True, zero_rows=cz, want_had=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(qr.cpu().numpy(), codes_r.cpu().numpy())
    np.testing.assert_array_equal(sr.cpu().numpy(), scales_r.cpu().numpy())
    np.testing.assert_array_equal(qc.cpu().numpy(), codes_c.cpu().numpy())
    np.testing.assert_array_equal(sc.cpu().numpy(), scales_c.cpu().numpy())
    for had, codes, scales in ((had_r, qr, sr), (had_c, qc, sc)):
        oc, osc = O.quantize_mxfp4(had.cpu().numpy())
        np.testing.assert_array_equal(scales.cpu().numpy(), osc)
        np.testing.assert_array_equal(codes.cpu().numpy(), O.pack_codes(oc))
    xs = x.copy()
    if masks:
        xs[np.asarray(rz)] = 0.0
        assert rel_fro(had_r.cpu().numpy(), O.iht_dense(xs)) <= TOL_HAD
        xt = x.T.copy()
        xt[np.asarray(cz)] = 0.0
        assert rel_fro(had_c.cpu().numpy(), O.iht_dense(xt)) <= TOL_HAD
        # raw OE slices: the extracted rows / columns of T, bf16 exact
        np.testing.assert_array_equal(slr.float().cpu().numpy(), x[np.asarray(rz)])
        np.testing.assert_array_equal(slc.float().cpu().numpy(), x.T[np.asarray(cz)])


def test_iht_quant_extreme_magnitudes():
    rng = np.random.default_rng(5)
    R, K = 64, 256
    x = rng.standard_normal((R, K)).astype(np.float32)
    scale = np.float32(2.0) ** rng.integers(-140, 120, size=(R, 1)).astype(np.float32)
    x = (x * scale).astype(np.float32)
    x[3] = 0.0
    x[4, :] = 0.0
    x[4, 7] = np.float32(1e-45)        # smallest subnormal
    x[5] = np.float32(3e38) * np.sign(x[5])
    t = dev_f32(x)
    codes, scales, had = ah.debug_iht_quant(t, want_had=True)
    spec = O.fwht_fp32_spec(x)
    finite = np.isfinite(spec).all(axis=1)
    oc, osc = O.quantize_mxfp4(np.where(np.isfinite(spec), spec, 0))
    np.testing.assert_array_equal(scales.cpu().numpy()[finite], osc[finite])
    np.testing.assert_array_equal(codes.cpu().numpy()[finite], O.pack_codes(oc)[finite])


def _extreme_bf16_rows(R, K, seed):
    # bf16 rows whose per-row scales sweep the whole bf16 exponent range (2^-133 ... 2^120), plus
    # zero rows, a row holding only the smallest bf16 subnormal, and rows with one near-max
    # element per 32-block (Hadamard outputs ~2^125.5: scale exponent e = 123, the quantiser's
    # e > 120 fallback); the low rows take its e < -100 fallback
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((R, K)).astype(np.float64)
    ex = np.round(np.linspace(-133, 118, R))
    x *= np.exp2(ex)[:, None]
    x[3] = 0.0
    x[4] = 0.0
    x[4, 7] = 2.0 ** -133
    # (rows 5 and 6 put theirs in different columns, so that no 32-block of either orientation
    # holds two of them: the transform of finite inputs must stay finite, include/adahop.h)
    for r, c0 in ((5, 0), (6, 16)):
        x[r] = 0.0
        x[r, c0::32] = 3.3e38 * np.where(rng.standard_normal(K // 32) > 0, 1.0, -1.0)
    return O.round_bf16(x.astype(np.float32))


@pytest.mark.parametrize("k_strided", [False, True])
def test_quant_tc_bf16_extreme_magnitudes_production_path(k_strided):
    # The tensor-core quantiser on bf16 inputs (the production path of every bf16 operand): the
    # fp32 Hadamard dump (debug variant) fixes the quantiser's input; the PRODUCTION variant (no
    # dump: fused c * 2^-e multiply, fallbacks for e > 120 / e < -100) must give the oracle's
    # codes and scales of that input bit for bit (SURVEY c19 protocol (a)).
    R, K = 256, 512
    x = _extreme_bf16_rows(R, K, 21)
    t = dev_bf16(x.T.copy() if k_strided else x)
    _, _, had = ah.debug_iht_quant(t, k_strided=k_strided, want_had=True)
    codes, scales, _ = ah.debug_iht_quant(t, k_strided=k_strided, want_had=False)
    torch.cuda.synchronize()
    had = had.cpu().numpy()
    assert np.isfinite(had).all()
    oc, osc = O.quantize_mxfp4(had)
    np.testing.assert_array_equal(scales.cpu().numpy(), osc)
    np.testing.assert_array_equal(codes.cpu().numpy(), O.pack_codes(oc))
    assert osc.max() >= 127 + 121 and osc[osc != 127].min() <= 127 - 101   # both fallbacks exercised
    # the Hadamard output itself: within 1e-6 of the exact transform, per row (rows of normal
    # fp32 magnitude; subnormal outputs carry fewer significant bits by construction)
    ref = O.iht_dense(x)
    big = np.abs(ref).max(1) >= 2.0 ** -100
    err = np.linalg.norm(had - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
    assert np.all(err[big] <= TOL_HAD)


def test_quant_dual_bf16_extreme_magnitudes_production_path():
    # the dual-orientation production launch (row + column layouts of one tensor in one pass) at
    # the same magnitudes, against the oracle quantiser of each orientation's Hadamard dump
    R, C = 256, 512
    x = _extreme_bf16_rows(R, C, 22)
    t = dev_bf16(x)
    qr, sr, qc, sc = ah.debug_quant_dual(t)
    _, _, had_r = ah.debug_iht_quant(t, want_had=True)
    _, _, had_c = ah.debug_iht_quant(t, k_strided=True, want_had=True)
    torch.cuda.synchronize()
    for had, q, sc_ in ((had_r, qr, sr), (had_c, qc, sc)):
        assert torch.isfinite(had).all()
        oc, osc = O.quantize_mxfp4(had.cpu().numpy())
        np.testing.assert_array_equal(sc_.cpu().numpy(), osc)
        np.testing.assert_array_equal(q.cpu().numpy(), O.pack_codes(oc))


# ======================================================================= FOID
@pytest.mark.parametrize("k_strided", [False, True])
@pytest.mark.parametrize("R,K,k,probe", [(5000, 128, 64, 64), (300, 96, 8, 64), (2048, 64, 256, 64),
                                          (4100, 256, 16, 32), (50, 32, 64, 64), (16384, 512, 64, 64),
                                          (16384, 64, 256, 64), (32768, 64, 256, 64), (9000, 160, 64, 96),
                                          (7, 64, 64, 64)])
def test_foid_index_sets_bitexact(R, K, k, probe, k_strided):
    # 32768 rows: 8 select blocks and their merge; probe 96 > 64 takes the generic key path;
    # R = 7 < k clamps; a key tie across select blocks
    x, planted = synth.operand(R, K, "R", "X", case_id=R + k, count=min(5, R))
    x[min(10, R - 1)] = x[min(11, R - 2)]          # an exact key tie
    if R > 8192:
        x[R - 3] = x[5]                            # a tie across the cluster's CTAs
    xin = x.T.copy() if k_strided else x
    idx, keys = ah.debug_foid(dev_bf16(xin), k=k, probe=probe, k_strided=k_strided)
    want_keys = O.foid_keys(x, probe)
    np.testing.assert_array_equal(keys.cpu().numpy().view(np.uint64), want_keys.view(np.uint64))
    np.testing.assert_array_equal(idx.cpu().numpy(), O.foid_indices(x, k, probe))
    assert set(planted.rows) <= set(idx.cpu().numpy().tolist())


def test_foid_row_limit_is_reported():
    x = torch.zeros((65537, 64), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(ah.AdahopError) as e:
        ah.debug_foid(x, k=8)
    assert "unsupported" in str(e.value)


@pytest.mark.parametrize("k_strided", [False, True])
@pytest.mark.parametrize("k", [64, 256])
def test_foid_65536_rows_bitexact(k, k_strided):
    # 65536 stored rows (e.g. 64k tokens per GPU for an OE on the token dimension): 16 select
    # blocks whose survivors the last block merges (PAPER P:760 FOID, DESIGN R5 keys and ties)
    R, K = 65536, 64
    x, planted = synth.operand(R, K, "R", "X", case_id=R + k, count=12)
    x[70000 % R] = x[123]                          # an exact key tie across select blocks
    xin = x.T.copy() if k_strided else x
    idx, keys = ah.debug_foid(dev_bf16(xin), k=k, k_strided=k_strided)
    np.testing.assert_array_equal(keys.cpu().numpy().view(np.uint64), O.foid_keys(x).view(np.uint64))
    np.testing.assert_array_equal(idx.cpu().numpy(), O.foid_indices(x, k))
    assert set(planted.rows) <= set(idx.cpu().numpy().tolist())


def test_oe_left_on_65536_tokens_layer_sampled():
    # dgrad OE-Left (RN: G_Y row-wise) with the extracted rows chosen among 65536 tokens: FOID over
    # 65536 rows, the row mask of the dual quantiser beyond the old 32768-row bitmap, the outlier
    # GEMM and the fused scatter; sampled against the oracle (all extracted rows included)
    T, d_in, d_out = 65536, 256, 512
    x, _ = synth.operand(T, d_in, "C", "X", case_id=961)
    w, _ = synth.operand(d_out, d_in, "N", "W", case_id=962)
    gy, planted = synth.operand(T, d_out, "R", "GY", case_id=963)
    strats = ("IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT")
    p = ah.Params(oe_k=64)
    y, gx, gw = ah.linear_layer(dev_bf16(x), dev_bf16(w), dev_bf16(gy), strats, p, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    idx = O.foid_indices(gy, 64)
    # 0.1 % of 65536 tokens = 66 planted rows > k = 64: every extracted row is a planted one
    assert len(planted.rows) > 64 and set(idx.tolist()) <= set(int(r) for r in planted.rows)
    rows = np.concatenate([rng.integers(0, T, 1500), idx])
    cols = rng.integers(0, d_in, rows.size)
    a_store, b_store = O.path_operands("dgrad", x=x, w=w, gy=gy)
    ref = O.sampled_entries(np.ascontiguousarray(a_store), np.ascontiguousarray(b_store), "OE_LEFT_IHT", rows, cols)
    assert rel_fro(gx.cpu().numpy()[rows, cols], ref) <= TOL_OUT
    # the wgrad (K = 65536 tokens) and fwd of the same call
    for path, got, s in (("fwd", y, "IHT"), ("wgrad", gw, "OE_RIGHT_IHT")):
        a_store, b_store = O.path_operands(path, x=x, w=w, gy=gy)
        r_ = rng.integers(0, got.shape[0], 1500)
        c_ = rng.integers(0, got.shape[1], 1500)
        ref = O.sampled_entries(np.ascontiguousarray(a_store), np.ascontiguousarray(b_store), s, r_, c_)
        assert rel_fro(got.cpu().numpy()[r_, c_], ref) <= TOL_OUT, path


# ======================================================================= MXFP4 GEMM
def _rand_mx(R, K, rng):
    codes = rng.integers(0, 16, size=(R, K), dtype=np.uint8)
    scales = rng.integers(127 - 6, 127 + 6, size=(R, K // 32), dtype=np.uint8)
    return codes, scales


def test_gemm_mxf4_one_hot_layout():
    M, N, K = 256, 256, 512
    for (r, n, k, ca, cb, ea, eb) in [(0, 0, 0, 2, 2, 127, 127), (5, 17, 33, 7, 3, 129, 120),
                                      (130, 255, 511, 15, 9, 127, 140), (255, 128, 300, 4, 4, 100, 150)]:
        a = np.zeros((M, K), np.uint8)
        b = np.zeros((N, K), np.uint8)
        a[r, k] = ca
        b[n, k] = cb
        sa = np.full((M, K // 32), 127, np.uint8)
        sb = np.full((N, K // 32), 127, np.uint8)
        sa[r, k // 32] = ea
        sb[n, k // 32] = eb
        c = ah.debug_gemm_mxf4(*(torch.from_numpy(v).to(DEV) for v in (O.pack_codes(a), sa, O.pack_codes(b), sb)))
        c = c.cpu().numpy()
        want = O.dequantize_mxfp4(a, sa) @ O.dequantize_mxfp4(b, sb).T
        nz = np.argwhere(c != 0)
        np.testing.assert_array_equal(c, want)
        assert len(nz) <= 1


# the last three: long K with few 256 x 256 tiles -> split-K clusters (4 pairs: 8 and 6 ragged
# tiles; 2 pairs: 24 tiles), partials summed across the cluster in distributed shared memory
@pytest.mark.parametrize("M,N,K", [(256, 128, 256), (300, 200, 544), (128, 384, 2048), (1000, 520, 1024),
                                   (512, 1024, 8192), (300, 700, 8192), (768, 2048, 8192)])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_gemm_mxf4_random_vs_oracle(M, N, K, out):
    rng = np.random.default_rng(M + N + K)
    ca, sa = _rand_mx(M, K, rng)
    cb, sb = _rand_mx(N, K, rng)
    ops = [torch.from_numpy(v).to(DEV) for v in (O.pack_codes(ca), sa, O.pack_codes(cb), sb)]
    c32 = ah.debug_gemm_mxf4(*ops, out_dtype=torch.float32).cpu().numpy()
    want = O.dequantize_mxfp4(ca, sa) @ O.dequantize_mxfp4(cb, sb).T
    assert rel_fro(c32, want) <= 1e-5
    if out == "bf16":
        c16 = ah.debug_gemm_mxf4(*ops, out_dtype=torch.bfloat16).float().cpu().numpy()
        np.testing.assert_array_equal(c16, O.round_bf16(c32).astype(np.float32))


# ======================================================================= end-to-end GEMM
STRATS = ["IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT", "BF16"]


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("a_ks,b_ks", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_adahop_gemm_vs_oracle(strategy, a_ks, b_ks):
    M, N, K, k = 384, 320, 512, 16
    a, _ = synth.operand(M, K, "R", "X", case_id=31, count=4)          # A_store rows planted
    b, _ = synth.operand(N, K, "R", "W", case_id=32, count=3)          # B_store rows = B columns
    ta = dev_bf16(a.T.copy() if a_ks else a)
    tb = dev_bf16(b.T.copy() if b_ks else b)
    p = ah.Params(oe_k=k)
    c = ah.gemm(ta, a_ks, tb, b_ks, M, N, K, strategy, p, out_dtype=torch.float32)
    cb16 = ah.gemm(ta, a_ks, tb, b_ks, M, N, K, strategy, p, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    ref, parts = O.adahop_matmul(a, b, strategy, k=k, return_parts=True)
    got = c.cpu().numpy()
    assert rel_fro(got, ref) <= TOL_OUT
    # bf16 output = RN_bf16(fp32 output): same accumulator, epilogue-only conversion
    np.testing.assert_array_equal(cb16.float().cpu().numpy(), O.round_bf16(got).astype(np.float32))
    if strategy in ("OE_LEFT_IHT", "OE_RIGHT_IHT"):
        idx = parts["idx"]
        sel = got[idx, :] if strategy == "OE_LEFT_IHT" else got[:, idx]
        # disjoint support: the extracted rows/cols carry exactly the BF16 outlier product
        assert rel_fro(sel, parts["c_out"]) <= 1e-5


@pytest.mark.parametrize("a_ks,b_ks", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(640, 520, 4128), (288, 1000, 544)])
def test_adahop_gemm_bf16_pair_kernel_vs_oracle(M, N, K, a_ks, b_ks):
    """The Lv2 CC product on CTA pairs (kind::f16, M = 256 tiles; K >= 4096: overlapping
    accumulators): K-major and MN-major operands, ragged M / N / K, bf16 = RN(fp32) output."""
    a, _ = synth.operand(M, K, "C", "X", case_id=M + K + a_ks, count=3)
    b, _ = synth.operand(N, K, "C", "W", case_id=N + K + b_ks, count=3)
    ta = dev_bf16(a.T.copy() if a_ks else a)
    tb = dev_bf16(b.T.copy() if b_ks else b)
    c = ah.gemm(ta, a_ks, tb, b_ks, M, N, K, "BF16", out_dtype=torch.float32)
    cb16 = ah.gemm(ta, a_ks, tb, b_ks, M, N, K, "BF16", out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    ref = O.adahop_matmul(a, b, "BF16")
    got = c.cpu().numpy()
    assert rel_fro(got, ref) <= 1e-5   # bf16 operands exact, fp32 accumulation
    np.testing.assert_array_equal(cb16.float().cpu().numpy(), O.round_bf16(got).astype(np.float32))


@pytest.mark.parametrize("strategy", ["IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT"])
def test_adahop_gemm_splitk_vs_oracle(strategy):
    """Long-K GEMM with 4 output tiles: split-K over a cluster of 4 pairs; the outlier entries
    are patched by the CTA that sums their column slice."""
    M, N, K, k = 512, 384, 8192, 16
    a, _ = synth.operand(M, K, "R", "X", case_id=33, count=4)
    b, _ = synth.operand(N, K, "R", "W", case_id=34, count=3)
    p = ah.Params(oe_k=k)
    c = ah.gemm(dev_bf16(a), 0, dev_bf16(b), 0, M, N, K, strategy, p, out_dtype=torch.float32)
    c2 = ah.gemm(dev_bf16(a), 0, dev_bf16(b), 0, M, N, K, strategy, p, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref, parts = O.adahop_matmul(a, b, strategy, k=k, return_parts=True)
    got = c.cpu().numpy()
    assert rel_fro(got, ref) <= TOL_OUT
    np.testing.assert_array_equal(c2.cpu().numpy().view(np.uint32), got.view(np.uint32))   # fixed-order sum
    if strategy != "IHT":
        idx = parts["idx"]
        sel = got[idx, :] if strategy == "OE_LEFT_IHT" else got[:, idx]
        assert rel_fro(sel, parts["c_out"]) <= 1e-5


def test_adahop_gemm_k_clamp_and_k0():
    M, N, K = 40, 72, 96
    a, _ = synth.operand(M, K, "N", "X", case_id=41)
    b, _ = synth.operand(N, K, "N", "W", case_id=42)
    for strategy, k in (("OE_LEFT_IHT", 100), ("OE_RIGHT_IHT", 100), ("OE_LEFT_IHT", 0)):
        c = ah.gemm(dev_bf16(a), 0, dev_bf16(b), 0, M, N, K, strategy, ah.Params(oe_k=k), out_dtype=torch.float32)
        ref = O.adahop_matmul(a, b, strategy, k=k)
        assert rel_fro(c.cpu().numpy(), ref) <= (1e-5 if k == 100 else TOL_OUT)


def test_adahop_gemm_deterministic():
    M, N, K = 512, 384, 1024
    a, _ = synth.operand(M, K, "R", "X", case_id=51)
    b, _ = synth.operand(N, K, "C", "W", case_id=52)
    ta, tb = dev_bf16(a), dev_bf16(b)
    outs = [ah.gemm(ta, 0, tb, 0, M, N, K, "OE_RIGHT_IHT", out_dtype=torch.float32).cpu().numpy() for _ in range(3)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o.view(np.uint32), outs[0].view(np.uint32))


# ======================================================================= linear paths, 9 pairs
PAIRS = [(x, g) for x in "RCN" for g in "RCN"]


@pytest.mark.parametrize("level", [1, 2])
@pytest.mark.parametrize("path", ["fwd", "dgrad", "wgrad"])
def test_linear_paths_all_pairs(path, level):
    T, d_in, d_out = 512, 384, 256
    for i, (pa, pb) in enumerate(PAIRS):
        # choose tensor patterns so that the FED pair of this path is (pa, pb)
        t = O.transpose_pattern
        if path == "fwd":
            px, pw, pg = pa, t(pb), "N"
        elif path == "dgrad":
            px, pw, pg = "N", pb, pa
        else:
            px, pw, pg = pb, "N", t(pa)
        x, _ = synth.operand(T, d_in, px, "X", case_id=100 + i)
        w, _ = synth.operand(d_out, d_in, pw, "W", case_id=200 + i)
        gy, _ = synth.operand(T, d_out, pg, "GY", case_id=300 + i)
        assert O.fed_patterns(path, px, pw, pg) == (pa, pb)
        strategy = O.strategy_for_pair(pa, pb, level)
        assert ah.strategy_for_pair(pa, pb, level) == strategy
        p = ah.Params(oe_k=16, level=level)
        got = ah.linear(path, strategy, x=dev_bf16(x), w=dev_bf16(w), gy=dev_bf16(gy), params=p,
                        out_dtype=torch.float32).cpu().numpy()
        ref = O.linear(path, strategy, x=x, w=w, gy=gy, k=16)
        err = rel_fro(got, ref)
        assert err <= TOL_OUT, (path, pa + pb, strategy, err)


# ======================================================================= calibration
@pytest.mark.parametrize("shape", [(256, 256), (2048, 512), (512, 4096)])
def test_calibration_patterns_and_cv(shape):
    rows, cols = shape
    for i, p in enumerate("RCN"):
        t, _ = synth.operand(rows, cols, p, "GY", case_id=60 + i)
        pat, cvr, cvc = ah.calibrate(dev_bf16(t))
        orow, ocol = O.cv_row_col(t)
        assert abs(cvr - orow) <= 1e-9 * max(1, orow) and abs(cvc - ocol) <= 1e-9 * max(1, ocol)
        assert pat == O.classify(t) == p


# ======================================================================= full-size sampled parity
@pytest.mark.slow
@pytest.mark.parametrize("path,strategy,pats", [("fwd", "IHT", ("C", "N", "N")),
                                                ("wgrad", "OE_RIGHT_IHT", ("C", "N", "C")),
                                                ("dgrad", "OE_LEFT_IHT", ("N", "N", "R"))])
def test_full_size_llama1b_sampled(path, strategy, pats):
    T, d_in, d_out = 16384, 2048, 2048
    px, pw, pg = pats
    x, _ = synth.operand(T, d_in, px, "X", case_id=71)
    w, _ = synth.operand(d_out, d_in, pw, "W", case_id=72)
    gy, _ = synth.operand(T, d_out, pg, "GY", case_id=73)
    got = ah.linear(path, strategy, x=dev_bf16(x), w=dev_bf16(w), gy=dev_bf16(gy), out_dtype=torch.float32)
    got = got.cpu().numpy()
    a_store, b_store = O.path_operands(path, x=x, w=w, gy=gy)
    rng = np.random.default_rng(9)
    rows = rng.integers(0, got.shape[0], 3000)
    cols = rng.integers(0, got.shape[1], 3000)
    if strategy != "IHT":
        oe_store = a_store if strategy == "OE_LEFT_IHT" else b_store
        idx = O.foid_indices(np.ascontiguousarray(oe_store), 64)
        extra = rng.integers(0, got.shape[1 if strategy == "OE_LEFT_IHT" else 0], len(idx))
        if strategy == "OE_LEFT_IHT":
            rows, cols = np.concatenate([rows, idx]), np.concatenate([cols, extra])
        else:
            rows, cols = np.concatenate([rows, extra]), np.concatenate([cols, idx])
    ref = O.sampled_entries(np.ascontiguousarray(a_store), np.ascontiguousarray(b_store), strategy, rows, cols)
    assert rel_fro(got[rows, cols], ref) <= TOL_OUT


# ======================================================================= layer step (dual quant)
LAYER_STRATS = [("IHT", "IHT", "OE_RIGHT_IHT"), ("IHT", "OE_LEFT_IHT", "OE_LEFT_IHT"),
                ("OE_LEFT_IHT", "OE_RIGHT_IHT", "OE_RIGHT_IHT"), ("OE_RIGHT_IHT", "IHT", "BF16"),
                ("BF16", "BF16", "IHT")]


@pytest.mark.parametrize("shape", [(640, 384, 256), (544, 352, 224), (512, 160, 96)])
@pytest.mark.parametrize("strats", LAYER_STRATS)
def test_linear_layer_matches_paths_and_oracle(strats, shape):
    T, d_in, d_out = shape
    x, _ = synth.operand(T, d_in, "C", "X", case_id=401)
    w, _ = synth.operand(d_out, d_in, "N", "W", case_id=402)
    gy, _ = synth.operand(T, d_out, "R", "GY", case_id=403)
    p = ah.Params(oe_k=16)
    xd, wd, gd = dev_bf16(x), dev_bf16(w), dev_bf16(gy)
    y, gx, gw = ah.linear_layer(xd, wd, gd, strats, p, out_dtype=torch.float32)
    # identical (bitwise) to the three per-path calls: same quantiser arithmetic, one read
    y1 = ah.linear_fwd(xd, wd, strats[0], p, out_dtype=torch.float32)
    gx1 = ah.linear_dgrad(gd, wd, strats[1], p, out_dtype=torch.float32)
    gw1 = ah.linear_wgrad(gd, xd, strats[2], p, out_dtype=torch.float32)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy().view(np.uint32), y1.cpu().numpy().view(np.uint32))
    # dgrad: bitwise, except that with OE-Left the layer call accumulates the outlier product
    # G_Y[S, :] W in W's quant pass and the per-path call in a BF16 GEMM (DESIGN R15): the k
    # extracted rows of G_X agree to rounding
    a, b = gx.cpu().numpy(), gx1.cpu().numpy()
    diff = a.view(np.uint32) != b.view(np.uint32)
    if strats[1] == "OE_LEFT_IHT":
        assert len(np.unique(np.nonzero(diff)[0])) <= 16
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6 * np.abs(b).max())
    else:
        assert not diff.any()
    # wgrad: the MXFP4 part is bitwise equal; with OE the layer call accumulates the outlier product
    # in a quant pass (G_Y's for OE-Right, X's for OE-Left) and the per-path call in a split-K BF16
    # GEMM, two fp32 summation orders of the same product (DESIGN R15), so the extracted
    # columns / rows agree to rounding
    a, b = gw.cpu().numpy(), gw1.cpu().numpy()
    diff = a.view(np.uint32) != b.view(np.uint32)
    if strats[2] in ("OE_RIGHT_IHT", "OE_LEFT_IHT"):
        axis = 1 if strats[2] == "OE_RIGHT_IHT" else 0   # extracted columns / rows of G_W
        assert len(np.unique(np.nonzero(diff)[axis])) <= 16   # at most the k = 16 extracted ones
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6 * np.abs(b).max())
    else:
        assert not diff.any()
    for path, got, s in (("fwd", y, strats[0]), ("dgrad", gx, strats[1]), ("wgrad", gw, strats[2])):
        ref = O.linear(path, s, x=x, w=w, gy=gy, k=16)
        assert rel_fro(got.cpu().numpy(), ref) <= TOL_OUT, (path, s)


def test_gemm_kernel_alone_matches_debug_gemm():
    # adahop_debug_gemm_mxf4_tcsf (the kernel alone, scales already in the tcgen05 layout) equals the
    # canonical-layout debug GEMM when every scale byte is the same (layout-independent scales)
    M, N, K = 384, 640, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    for e in (120, 127, 131):
        sa = torch.full((M, K // 32), e, dtype=torch.uint8, device="cuda")
        sb = torch.full((N, K // 32), e, dtype=torch.uint8, device="cuda")
        ref = ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.float32)
        ea = torch.full((ah.debug_sf_bytes(M, K),), e, dtype=torch.uint8, device="cuda")
        eb = torch.full((ah.debug_sf_bytes(N, K),), e, dtype=torch.uint8, device="cuda")
        got = ah.debug_gemm_mxf4_tcsf(a, ea, b, eb, torch.empty((M, N), dtype=torch.float32, device="cuda"))
        torch.cuda.synchronize()
        assert torch.equal(got, ref)


def test_calibrate_batch_equals_per_tensor_calls():
    # adahop_calibrate_batch: the same partition and reduction order as adahop_calibrate, so the CV
    # sums, CVs and patterns are bitwise equal; 35 tensors exercise the 32-job chunking, ragged shapes
    rng = np.random.default_rng(11)
    shapes = [(int(rng.integers(1, 700)), int(rng.integers(1, 900))) for _ in range(33)] + [(2048, 512), (384, 4096)]
    pats = "RCN"
    ts = [dev_bf16(synth.operand(r, c, pats[i % 3], "X", case_id=700 + i)[0]) for i, (r, c) in enumerate(shapes)]
    ws = torch.empty(ah.calibrate_batch_workspace_bytes([t.shape for t in ts]), dtype=torch.uint8, device="cuda")
    cv = torch.full((len(ts), 4), -1.0, dtype=torch.float64, device="cuda")
    pat = torch.full((len(ts),), 255, dtype=torch.uint8, device="cuda")
    ah.calibrate_batch_async(ts, ws, cv, pat)
    one_ws = torch.empty(max(ah.calibrate_workspace_bytes(*t.shape) for t in ts), dtype=torch.uint8, device="cuda")
    cv1 = torch.empty_like(cv)
    pat1 = torch.empty_like(pat)
    for i, t in enumerate(ts):
        ah.calibrate_async(t, one_ws, cv1[i], pat1[i:i + 1])
    torch.cuda.synchronize()
    assert torch.equal(cv.view(torch.int64), cv1.view(torch.int64))
    assert torch.equal(pat, pat1)
    for i, t in enumerate(ts):   # and the oracle's decision on the planted ones
        if min(shapes[i]) >= 64:
            assert "NRC"[int(pat[i])] == O.classify(t.float().cpu().numpy().astype(np.float64)), i
