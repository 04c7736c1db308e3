"""GPU parity: quantisation kernels vs the oracle and the reference's golden fixtures (bit-exact)."""

import hashlib
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2402_13533_b200 as qa

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_quantize_rows_matches_reference_golden(golden_dir):
    g = np.load(os.path.join(golden_dir, "quant_cases.npz"))
    names = sorted({k.split("__")[0] for k in g.files})
    for name in names:
        w = g[f"{name}__w"]
        for bits in (4, 8):
            q = qa.quantize_rows(w, bits)
            assert _np(q.codes).tobytes() == g[f"{name}__b{bits}__codes"].tobytes(), (name, bits)
            assert _np(q.scale).tobytes() == g[f"{name}__b{bits}__scale"].tobytes(), (name, bits)
            assert _np(q.offset).tobytes() == g[f"{name}__b{bits}__offset"].tobytes(), (name, bits)
            ref = O.quantize_rows(w, bits)
            assert _np(q.rowsum).astype(np.int64).tolist() == ref.rowsum().tolist()
            deq = qa.dequantize_rows(q, torch.float32)
            assert _np(deq).tobytes() == g[f"{name}__b{bits}__deq"].astype(np.float32).tobytes(), (name, bits)


def test_config1_weight_and_token_codes_bit_exact(golden_dir):
    g = np.load(os.path.join(golden_dir, "config1.npz"))
    W = O.seeded_random(1024, 1024, 1, std=0.02)
    X = O.seeded_random(512, 1024, 2)
    qw, qw4, qx = qa.quantize_rows(W, 8), qa.quantize_rows(W, 4), qa.quantize_rows(X, 8)
    assert _digest(_np(qw.codes)) == str(g["qw_codes_digest"])
    assert _digest(_np(qw4.codes)) == str(g["qw4_codes_digest"])
    assert _digest(_np(qx.codes)) == str(g["qx_codes_digest"])
    assert _np(qw.scale).tobytes() == g["qw_scale"].tobytes()
    assert _np(qx.offset).tobytes() == g["qx_offset"].tobytes()


@pytest.mark.parametrize("shape", [(4096, 4096), (333, 11008), (1, 7), (17, 1031), (64, 28672)])
def test_bf16_activation_codes_bit_exact_large(shape):
    torch.manual_seed(shape[0] * 7 + shape[1])
    x = torch.randn(shape, device="cuda").to(torch.bfloat16)
    xf = x.float().cpu().numpy()
    for bits in (8, 4):
        q = qa.quantize_rows(x, bits)
        ref = O.quantize_rows(xf, bits)
        got = _np(q.codes)
        if got.tobytes() != ref.codes.tobytes():
            bad = np.argwhere(got != ref.codes)
            raise AssertionError(f"{len(bad)} code mismatches, first {bad[:5].tolist()}")
        assert _np(q.scale).tobytes() == ref.scale.tobytes()
        assert _np(q.offset).tobytes() == ref.offset.tobytes()


def test_tie_and_near_tie_rows(golden_dir):
    g = np.load(os.path.join(golden_dir, "quant_cases.npz"))
    for name in ("ties", "nearties"):
        q = qa.quantize_rows(g[f"{name}__w"], 8)
        assert _np(q.codes).tobytes() == g[f"{name}__b8__codes"].tobytes()
    # synthetic near-tie stress: values placed within 1e-5 of half-steps of a 255-level grid
    rng = np.random.default_rng(0)
    k = rng.integers(0, 255, size=(64, 4096)).astype(np.float64) + 0.5
    w = (k + rng.uniform(-3e-5, 3e-5, size=k.shape)).astype(np.float32)
    w[:, 0], w[:, 1] = 0.0, 255.0
    q = qa.quantize_rows(w, 8)
    assert _np(q.codes).tobytes() == O.quantize_rows(w, 8).codes.tobytes()


def test_kats_and_errors():
    q = qa.quantize_rows(np.array([[0.0, 1.0, 2.0, 3.0]], np.float32), 8)
    assert _np(q.codes)[0].tolist() == [0, 85, 170, 255]
    q = qa.quantize_rows(np.full((3, 5), 2.5, np.float32), 8)
    assert not _np(q.codes).any() and not _np(q.scale).any()
    assert qa.quantize_rows(O.seeded_random(3, 7, 9), 4).codes.shape == (3, 4)
    with pytest.raises(qa.QuantError):
        qa.quantize_rows(np.array([[1.0, np.inf]], np.float32), 8)
    with pytest.raises(qa.QuantError):
        qa.quantize_rows(np.array([[np.nan, 1.0]], np.float32), 4)
    with pytest.raises(qa.QuantError):
        qa.quantize_rows(np.ones((2, 2), np.float32), 3)
    with pytest.raises(qa.QuantError):
        qa.quantize_rows(np.ones(4, np.float32), 8)
    w = O.seeded_random(8, 8, 3)
    q = qa.quantize_rows(w, 8)
    q2 = qa.quantize_rows(qa.dequantize_rows(q), 8)  # requantise fixed point (test_quant.py:39-44)
    assert _np(q2.codes).tobytes() == _np(q.codes).tobytes()


def test_dequantize_transposed_bf16():
    w = O.seeded_random(300, 200, 4, std=0.02)
    for bits in (4, 8):
        q = qa.quantize_rows(w, bits)
        ref = O.dequantize_rows(O.quantize_rows(w, bits)).astype(np.float32)
        got = _np(qa.dequantize_rows(q, torch.bfloat16, transpose=True).float())
        np.testing.assert_allclose(got, ref.T, rtol=2 ** -8, atol=0)


def test_roundtrip_bound_full_size():
    # size-independent property at config-2 activation size: |x - deq(Q(x))| <= scale/2 (test_quant.py:31-37)
    torch.manual_seed(1)
    x = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
    q = qa.quantize_rows(x, 8)
    deq = qa.dequantize_rows(q, torch.float32)
    err = (deq - x.float()).abs()
    bound = q.scale[:, None] / 2 + 1e-6
    assert bool((err <= bound).all())
    assert torch.equal(q.rowsum.long(), q.codes.long().sum(1))
