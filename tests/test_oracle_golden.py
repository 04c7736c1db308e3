"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by oracle/gen_golden.py)
and to the reference test-suite KATs (pkg/tests/test_quant.py, test_lowrank.py)."""

import hashlib
import os

import numpy as np
import pytest

import oracle as O


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_seeded_random_bit_identical(golden_dir):
    g = _load(golden_dir, "seeded_random.npz")
    for seed in (0, 1, 7919, 123456789):
        assert O.seeded_random(3, 5, seed).tobytes() == g[f"g{seed}"].tobytes()
        got = O.seeded_random(2, 7, seed, dist="uniform", lo=-1, hi=2)
        assert got.tobytes() == g[f"u{seed}"].tobytes()


def _case_names(g):
    return sorted({k.split("__")[0] for k in g.files})


def test_quantize_rows_bit_exact_vs_reference(golden_dir):
    g = _load(golden_dir, "quant_cases.npz")
    names = _case_names(g)
    assert len(names) >= 10
    for name in names:
        w = g[f"{name}__w"]
        for bits in (4, 8):
            q = O.quantize_rows(w, bits)
            assert q.codes.tobytes() == g[f"{name}__b{bits}__codes"].tobytes(), (name, bits)
            assert q.scale.tobytes() == g[f"{name}__b{bits}__scale"].tobytes(), (name, bits)
            assert q.offset.tobytes() == g[f"{name}__b{bits}__offset"].tobytes(), (name, bits)
            np.testing.assert_array_equal(O.dequantize_rows(q), g[f"{name}__b{bits}__deq"])


def test_kats_from_reference_suite():
    # test_quant.py:26-29
    q = O.quantize_rows(np.array([[0.0, 1.0, 2.0, 3.0]], np.float32), 8)
    assert q.codes[0].tolist() == [0, 85, 170, 255]
    # test_quant.py:19-24 constant row -> scale 0, codes 0, exact dequant
    q = O.quantize_rows(np.full((3, 5), 2.5, np.float32), 8)
    assert not q.codes.any() and (q.scale == 0).all()
    np.testing.assert_array_equal(O.dequantize_rows(q, np.float32), np.full((3, 5), 2.5, np.float32))
    # test_quant.py:81-86 odd-column 4-bit pack 3x7 -> 3x4
    assert O.quantize_rows(O.seeded_random(3, 7, 9), 4).codes.shape == (3, 4)
    # test_quant.py:39-44 requantising the dequantised grid is a fixed point
    w = O.seeded_random(8, 8, 3)
    q = O.quantize_rows(w, 8)
    assert O.quantize_rows(O.dequantize_rows(q, np.float32), 8).codes.tobytes() == q.codes.tobytes()
    # test_quant.py:72-79 rejections
    with pytest.raises(O.OracleError):
        O.quantize_rows(np.array([[1.0, np.inf]], np.float32), 8)
    with pytest.raises(O.OracleError):
        O.quantize_rows(np.ones((2, 2), np.float32), 3)


def test_ties_round_away_from_zero(golden_dir):
    g = _load(golden_dir, "quant_cases.npz")
    q = O.quantize_rows(g["ties__w"], 8)
    # w = k/2 for k = 0..510 -> scale 1, v = k/2: halves round up
    expect = np.floor(np.arange(511) / 2 + 0.5).clip(0, 255).astype(np.uint8)
    assert q.codes[0].tolist() == expect.tolist()


def test_qmatmul_restatement(golden_dir):
    g = _load(golden_dir, "qmatmul_cases.npz")
    for bits in (4, 8):
        q = O.quantize_rows(g[f"b{bits}__w"], bits)
        np.testing.assert_allclose(O.qmatmul(q, g[f"b{bits}__x"]), g[f"b{bits}__qmatmul"], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(O.qmatmul_t(q, g[f"b{bits}__dy"]), g[f"b{bits}__qmatmul_t"], rtol=1e-13, atol=1e-15)


def test_dequant_identity_of_int32_epilogue():
    # A4: y1 = sx·sw·acc + sx·ow·Σcx + ox·sw·Σcw + K·ox·ow == qmatmul(qw, deq(qx))
    w = O.seeded_random(33, 64, 5, std=0.02)
    x = O.seeded_random(7, 64, 6)
    qw, qx = O.quantize_rows(w, 8), O.quantize_rows(x, 8)
    acc = O.int32_accumulators(qx, qw).astype(np.float64)
    sx, ox = qx.scale.astype(np.float64)[:, None], qx.offset.astype(np.float64)[:, None]
    sw, ow = qw.scale.astype(np.float64)[None, :], qw.offset.astype(np.float64)[None, :]
    y1 = sx * sw * acc + sx * ow * qx.rowsum()[:, None] + ox * sw * qw.rowsum()[None, :] + 64 * ox * ow
    np.testing.assert_allclose(y1, O.qmatmul(qw, O.dequantize_rows(qx)), rtol=1e-12, atol=1e-13)


def test_lora_as_two_core_tt_matches_reference_loralinear(golden_dir):
    g = _load(golden_dir, "lora_cases.npz")
    for bits in (4, 8):
        q = O.quantize_rows(g[f"b{bits}__w"], bits)
        shape, cores = O.lora_as_tt(g[f"b{bits}__down"].astype(np.float64), g[f"b{bits}__up"].astype(np.float64))
        x, dy = g[f"b{bits}__x"], g[f"b{bits}__dy"]
        # reference forward is qmatmul(x) + adapter (no act-quant in LoraLinear.forward)
        y = O.qmatmul(q, x) + O.tt_apply(x, cores)
        np.testing.assert_allclose(y, g[f"b{bits}__y"], rtol=1e-12, atol=1e-14)
        bw = O.qa_linear_backward(x, dy, q, cores)
        np.testing.assert_allclose(bw["dx"], g[f"b{bits}__dx"], rtol=1e-12, atol=1e-14)
        gd, gu = bw["dcores"]
        np.testing.assert_allclose(gd.reshape(-1, shape.ranks[1]).T, g[f"b{bits}__gdown"], rtol=1e-11, atol=1e-14)
        np.testing.assert_allclose(gu.reshape(shape.ranks[1], -1).T, g[f"b{bits}__gup"], rtol=1e-11, atol=1e-14)
        # merge: reference merges only dense bases; the quantised route is dequantise + W_t
        assert int(g[f"b{bits}__merge_q_refused"]) == 1
        dense_merge = g[f"b{bits}__w"].astype(np.float64) + O.tt_full(cores)
        np.testing.assert_allclose(dense_merge, g[f"b{bits}__merged_dense"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(O.qa_merge(q, cores), O.dequantize_rows(q) + O.tt_full(cores))


def test_config1_pins(golden_dir):
    g = _load(golden_dir, "config1.npz")
    W = O.seeded_random(1024, 1024, 1, std=0.02)
    X = O.seeded_random(512, 1024, 2)
    assert _digest(W) == str(g["w_digest"]) and _digest(X) == str(g["x_digest"])
    qw, qx, qw4 = O.quantize_rows(W, 8), O.quantize_rows(X, 8), O.quantize_rows(W, 4)
    assert _digest(qw.codes) == str(g["qw_codes_digest"])
    assert _digest(qw4.codes) == str(g["qw4_codes_digest"])
    assert _digest(qx.codes) == str(g["qx_codes_digest"])
    for a, k in ((qw.scale, "qw_scale"), (qw.offset, "qw_offset"), (qw4.scale, "qw4_scale"),
                 (qw4.offset, "qw4_offset"), (qx.scale, "qx_scale"), (qx.offset, "qx_offset")):
        assert a.tobytes() == g[k].tobytes(), k
    fw = O.qa_linear_forward(X[:16], qw, None)
    np.testing.assert_allclose(fw["y1"], g["y1_first16"], rtol=1e-12, atol=1e-13)
    bw = O.qa_linear_backward(X[:16], g["dy_first16"], qw, None)
    np.testing.assert_allclose(bw["dx"], g["dx_base_first16"], rtol=1e-12, atol=1e-13)


def _fd_check(shape, seed):
    rng = np.random.default_rng(seed)
    cores = [rng.standard_normal(shape.core_shape(k)) * 0.3 for k in range(shape.d)]
    x = rng.standard_normal((5, shape.K))
    tgt = rng.standard_normal((5, shape.N))
    dy = O.mse_grad(O.tt_apply(x, cores), tgt)
    grads = O.tt_core_grads(x, dy, cores)
    eps = 1e-6
    for k in range(shape.d):
        flat = cores[k].reshape(-1)
        for idx in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            old = flat[idx]
            flat[idx] = old + eps
            lp = O.mse_loss(O.tt_apply(x, cores), tgt)
            flat[idx] = old - eps
            lm = O.mse_loss(O.tt_apply(x, cores), tgt)
            flat[idx] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - grads[k].reshape(-1)[idx]) <= 1e-6 * max(1.0, abs(fd)), (k, idx)


def test_tt_core_grads_finite_differences():
    _fd_check(O.TTShape((2, 3, 2), (3, 2, 2), (1, 2, 3, 1)), 0)
    _fd_check(O.TTShape((1, 4, 8), (8, 2, 2), (1, 3, 3, 1)), 1)
    _fd_check(O.TTShape((2, 2), (3, 3), (1, 4, 1)), 2)


def test_tt_prefix_stages_compose_to_full():
    shape = O.TTShape((1, 4, 8), (8, 2, 2), (1, 3, 3, 1))
    rng = np.random.default_rng(3)
    cores = [rng.standard_normal(shape.core_shape(k)) for k in range(shape.d)]
    x = rng.standard_normal((4, shape.K))
    zs = O.tt_prefix(x, cores)
    u = zs[-1]  # [T, H, r, n_d]
    g = cores[-1]
    y2 = np.einsum("thbj,bij->thi", u, g[:, :, :, 0]).reshape(4, -1)
    np.testing.assert_allclose(y2, O.tt_apply(x, cores), rtol=1e-12)


def test_pinned_modes_cover_baseline_shapes():
    for n, k in ((4096, 4096), (11008, 4096), (4096, 11008), (8192, 8192), (1024, 8192),
                 (28672, 8192), (8192, 28672), (1024, 1024)):
        for r in (8, 16):
            s = O.tt_modes_for(n, k, r)
            assert s.N == n and s.K == k


def test_dp_mean_fixed_order():
    a = {"g": np.array([1.0, 2.0])}
    b = {"g": np.array([3.0, 6.0])}
    np.testing.assert_array_equal(O.dp_mean([a, b])["g"], [2.0, 4.0])


def test_staged_cpu_port_equals_materialised_oracle():
    for shape in (O.TTShape((1, 4, 8), (8, 2, 2), (1, 3, 3, 1)), O.TTShape((4, 16, 16), (4, 16, 16), (1, 8, 8, 1)),
                  O.TTShape((1, 32), (48, 1), (1, 4, 1))):
        rng = np.random.default_rng(7)
        cores = [rng.standard_normal(shape.core_shape(k)) for k in range(shape.d)]
        x = rng.standard_normal((9, shape.K))
        dy = rng.standard_normal((9, shape.N))
        np.testing.assert_allclose(O.tt_apply_staged(x, cores), O.tt_apply(x, cores), rtol=1e-10, atol=1e-10)
        dxa, grads = O.tt_backward_staged(x, dy, cores)
        np.testing.assert_allclose(dxa, O.tt_dx(dy, cores), rtol=1e-10, atol=1e-10)
        for g, gr in zip(grads, O.tt_core_grads(x, dy, cores)):
            np.testing.assert_allclose(g, gr, rtol=1e-10, atol=1e-9)
