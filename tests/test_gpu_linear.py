"""GPU parity of the quantised tensor-adapter linear (forward / backward-with-recompute / merge)
against the oracle, through the C ABI.

Tolerances: |got - want| <= rtol (|want| + rms(want)), reported by oracle.rel_err.
  exact : act/weight codes and the int32 accumulators
  1e-5  : fp32 outputs of fp32 arithmetic (y before bf16 rounding, merge in fp32)
  1e-2  : bf16 outputs and everything computed from bf16 operands (y, dx, adapter grads)
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2402_13533_b200 as qa
from paper_2402_13533_b200 import linear as L

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
TOL_BF16 = 1e-2
# adapter term y2 (probe output of the production GEMM): fp32-class — measured 5e-7..4e-5
TOL_Y2 = 1e-4
# adapter-core gradients. Generic stage kernels accumulate fp32 products of exact operands: measured
# <= 1.1e-6.  The fast family (first core input-only, last core output-only, LoRA) runs its dy pass on
# mma.sync with the intermediates Z2 / dZ2 / dZ1 as bf16 operands: measured 3.4e-3..6.1e-3 max-normalised,
# so it keeps the bf16 bar plus an average-case bar (Frobenius-relative) that a lost split term would break.
TOL_GRAD_GENERIC = 1e-4
TOL_GRAD_FAST = 1e-2
TOL_GRAD_FAST_RMS = 3e-3


def _np(t):
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()


def _case(N, K, T, bits, r, seed, spec=None, xdtype=torch.bfloat16):
    W = O.seeded_random(N, K, seed, std=0.02)
    Xf = O.seeded_random(T, K, seed + 1)
    x = torch.from_numpy(Xf).cuda().to(xdtype)
    xs = x.float().cpu().numpy()  # exact values the GPU sees
    q = qa.quantize_rows(W, bits)
    oq = O.quantize_rows(W, bits)
    if spec is None:
        spec = L.TTSpec.for_shape(N, K, r)
    shape = O.TTShape(spec.m, spec.n, spec.ranks)
    cores_np = O.tt_init_cores(shape, seed + 2, std=0.01)
    cores = [torch.from_numpy(c).cuda() for c in cores_np]
    return q, oq, x, xs, spec, cores, cores_np


CASES = [
    # (N, K, T, bits, r, spec)
    # generic TT path: config 1 (balanced modes), ragged / padded / int4 shapes
    (1024, 1024, 512, 8, 8, None),
    (1024, 1024, 512, 4, 8, None),
    (512, 768, 77, 8, 4, L.TTSpec((1, 2, 256), (48, 4, 4), (1, 4, 4, 1))),
    (320, 200, 130, 4, 3, L.TTSpec((4, 80), (20, 10), (1, 3, 1))),
    # fast TT family (first core input-only, last core output-only): pinned Llama modes and LoRA
    (256, 4096, 300, 8, 8, None),
    (4096, 1024, 200, 8, 16, None),
    (2048, 512, 97, 4, 8, None),
    (1024, 512, 150, 8, 8, L.TTSpec.lora(1024, 512, 8)),
    (768, 256, 64, 4, 16, L.TTSpec.lora(768, 256, 16)),
]


@pytest.mark.parametrize("N,K,T,bits,r,spec", CASES)
def test_forward_parity(N, K, T, bits, r, spec):
    q, oq, x, xs, spec, cores, cores_np = _case(N, K, T, bits, r, 11, spec)
    out = L.linear_forward(q, (spec, cores), x, debug=True)
    ref = O.qa_linear_forward(xs, oq, cores_np)
    acc = _np(out["acc"]).astype(np.int64)
    assert np.array_equal(acc, ref["acc"]), f"int32 accumulators differ at {np.argwhere(acc != ref['acc'])[:5]}"
    y2 = _np(out["y2"])
    e_y2 = O.rel_err(y2, ref["y2"])
    e_y1 = O.rel_err(_np(out["y_f32"]) - y2, ref["y1"])
    e_y = O.rel_err(_np(out["y_bf16"]), ref["y"])
    print(f"fwd {N}x{K} T={T} b{bits} r{r} {spec}: y1 {e_y1:.2e} y2 {e_y2:.2e} y {e_y:.2e}")
    assert e_y1 <= TOL_F32, e_y1
    assert e_y2 <= TOL_Y2, e_y2
    assert e_y <= TOL_BF16, e_y
    # production path (persistent GEMM, adapter folded in TMEM) against the oracle and the debug path
    y_prod = L.linear_forward(q, (spec, cores), x)
    assert O.rel_err(_np(y_prod), ref["y"]) <= TOL_BF16
    assert O.rel_err(_np(y_prod), _np(out["y_bf16"])) <= 2 ** -7


@pytest.mark.parametrize("N,K,T,bits,r,spec", CASES)
def test_backward_parity(N, K, T, bits, r, spec):
    q, oq, x, xs, spec, cores, cores_np = _case(N, K, T, bits, r, 21, spec)
    dy = torch.from_numpy(O.seeded_random(T, N, 99)).cuda().to(torch.bfloat16)
    dys = dy.float().cpu().numpy()
    dx, dcores, dx32 = L.linear_backward(q, (spec, cores), x, dy, debug=True)
    ref = O.qa_linear_backward(xs, dys, oq, cores_np)
    e32, e16 = O.rel_err(_np(dx32), ref["dx"]), O.rel_err(_np(dx), ref["dx"])
    eg = [O.rel_err(_np(g), gr) for g, gr in zip(dcores, ref["dcores"])]
    eg_rms = [O.rel_rms(_np(g), gr) for g, gr in zip(dcores, ref["dcores"])]
    print(f"bwd {N}x{K} T={T} b{bits} r{r} {spec}: dx32 {e32:.2e} dx {e16:.2e} grads "
          + " ".join(f"{e:.2e}/{f:.2e}" for e, f in zip(eg, eg_rms)))
    assert e32 <= TOL_BF16 and e16 <= TOL_BF16
    fast = spec.m[0] == 1 and spec.n[-1] == 1
    for k, (e, f) in enumerate(zip(eg, eg_rms)):
        if fast:
            assert e <= TOL_GRAD_FAST and f <= TOL_GRAD_FAST_RMS, (k, e, f)
        else:
            assert e <= TOL_GRAD_GENERIC, (k, e)


@pytest.mark.parametrize("N,K,T,bits,r,spec", CASES[4:])  # the fast TT family
def test_recompute_window_handoff_is_bit_identical(N, K, T, bits, r, spec):
    """qa_linear_forward_save + qa_linear_backward_saved (Z1 handed from the recompute-forward)
    gives exactly the gradients and dx of the backward that recomputes Z1 from x."""
    q, oq, x, xs, spec, cores, cores_np = _case(N, K, T, bits, r, 31, spec)
    dy = torch.from_numpy(O.seeded_random(T, N, 98)).cuda().to(torch.bfloat16)
    y_save, saved = L.linear_forward_saving(q, (spec, cores), x)
    assert saved is not None and saved.numel() > 0
    y_plain = L.linear_forward(q, (spec, cores), x)
    assert torch.equal(y_save, y_plain)
    dx_a, g_a = L.linear_backward(q, (spec, cores), x, dy, saved=saved)
    dx_b, g_b = L.linear_backward(q, (spec, cores), x, dy)
    assert torch.equal(dx_a, dx_b)
    for a, b in zip(g_a, g_b):
        assert torch.equal(a, b)
    # protocol level: TTLinear keeps the state for a backward on the same, unmodified x ...
    lin = L.TTLinear("w", L.QuantizedLinear("w.base", q), spec, [c.clone() for c in cores])
    grads = {}
    lin.forward(x)
    assert lin._saved is not None
    dx_c = lin.backward(x, dy, grads)
    assert torch.equal(dx_c, dx_b) and lin._saved is None
    # ... and recomputes when x changed in place after the forward
    lin.forward(x)
    x.mul_(1.0)
    assert lin._take_saved(x) is None


def test_base_only_paths_match_reference_functions():
    # qmatmul(act_quant=True) == qmatmul(qw, deq(Q(x))) (the paper's forward); the plain qmatmul / qmatmul_t /
    # qmatvec are the reference's own formulas (no activation quantisation) to fp32 accuracy
    W = O.seeded_random(384, 640, 5, std=0.02)
    X = O.seeded_random(200, 640, 6)
    dY = O.seeded_random(200, 384, 7)
    for bits in (4, 8):
        q, oq = qa.quantize_rows(W, bits), O.quantize_rows(W, bits)
        y = qa.qmatmul(q, torch.from_numpy(X).cuda(), act_quant=True)
        assert y.dtype == torch.float32
        want = O.qmatmul(oq, O.dequantize_rows(O.quantize_rows(X, 8)))
        assert O.rel_err(_np(y), want) <= TOL_F32
        y = qa.qmatmul(q, torch.from_numpy(X).cuda())
        assert O.rel_err(_np(y), O.qmatmul(oq, X)) <= TOL_F32
        yb = qa.qmatmul(q, torch.from_numpy(X).cuda().to(torch.bfloat16))
        assert O.rel_err(_np(yb), O.qmatmul(oq, O.to_bf16(X))) <= TOL_F32
        v = qa.qmatvec(q, torch.from_numpy(X[3]).cuda())
        assert v.shape == (384,) and O.rel_err(_np(v), O.qmatmul(oq, X[3])) <= TOL_F32
        dx = qa.qmatmul_t(q, torch.from_numpy(dY).cuda())
        assert O.rel_err(_np(dx), O.qmatmul_t(oq, dY)) <= TOL_F32
        # the training backward's bf16 path (QuantizedLinear.backward): deq(W) rounded to bf16
        dxb = L.QuantizedLinear("w", q).backward(None, torch.from_numpy(dY).cuda(), {})
        assert O.rel_err(_np(dxb), O.qmatmul_t(oq, dY)) <= TOL_BF16


def test_qmatmul_against_reference_golden(golden_dir):
    """quant.qmatmul / qmatmul_t outputs written by the reference itself (oracle/gen_golden.py), odd K = 13."""
    g = np.load(os.path.join(golden_dir, "qmatmul_cases.npz"))
    for bits in (4, 8):
        q = qa.quantize_rows(g[f"b{bits}__w"], bits)
        y = qa.qmatmul(q, torch.from_numpy(g[f"b{bits}__x"]).cuda())
        assert O.rel_err(_np(y), g[f"b{bits}__qmatmul"]) <= TOL_F32
        dx = qa.qmatmul_t(q, torch.from_numpy(g[f"b{bits}__dy"]).cuda())
        assert O.rel_err(_np(dx), g[f"b{bits}__qmatmul_t"]) <= TOL_F32
    c = np.load(os.path.join(golden_dir, "config1.npz"))
    W = O.seeded_random(1024, 1024, 1, std=0.02)
    X = O.seeded_random(512, 1024, 2)
    qw = qa.quantize_rows(W, 8)
    xd = qa.dequantize_rows(qa.quantize_rows(X, 8), torch.float32)[:16]
    assert O.rel_err(_np(qa.qmatmul(qw, xd)), c["y1_first16"]) <= TOL_F32
    assert O.rel_err(_np(qa.qmatmul_t(qw, torch.from_numpy(c["dy_first16"]).cuda())), c["dx_base_first16"]) <= TOL_F32
    with pytest.raises(qa.QuantError):
        qa.qmatmul(qw, torch.zeros(2, 1000, device="cuda"))
    with pytest.raises(qa.QuantError):
        qa.qmatmul_t(qw, torch.zeros(2, 1000, device="cuda"))


def test_lora_backend_is_drop_in_for_reference_loralinear(golden_dir):
    g = np.load(os.path.join(golden_dir, "lora_cases.npz"))
    for bits in (4, 8):
        base = L.QuantizedLinear("w.base", qa.quantize_rows(g[f"b{bits}__w"], bits))
        ad = L.LoraLinear("w", base, g[f"b{bits}__down"], g[f"b{bits}__up"])
        x = torch.from_numpy(g[f"b{bits}__x"].astype(np.float32)).cuda()
        dy = torch.from_numpy(g[f"b{bits}__dy"].astype(np.float32)).cuda()
        grads = {}
        dx = ad.backward(x, dy, grads)
        # the reference's own LoraLinear.backward outputs (transformer.py:310-318)
        assert set(grads) == {"w.down", "w.up"}
        assert O.rel_err(_np(dx), g[f"b{bits}__dx"]) <= TOL_BF16
        assert O.rel_err(_np(grads["w.down"]), g[f"b{bits}__gdown"]) <= TOL_BF16
        assert O.rel_err(_np(grads["w.up"]), g[f"b{bits}__gup"]) <= TOL_BF16
        # _accumulate semantics: a second backward adds
        ad.backward(x, dy, grads)
        assert O.rel_err(_np(grads["w.up"]), 2 * g[f"b{bits}__gup"]) <= TOL_BF16
        # forward = reference adapter + the paper's per-token act-quant of the base product
        y = ad.forward(x)
        oq = O.quantize_rows(g[f"b{bits}__w"], bits)
        _, cores = O.lora_as_tt(g[f"b{bits}__down"].astype(np.float64), g[f"b{bits}__up"].astype(np.float64))
        want = O.qa_linear_forward(x.cpu().numpy(), oq, cores)["y"]
        assert O.rel_err(_np(y), want) <= TOL_F32


@pytest.mark.parametrize("bits", [8, 4])
def test_merge_parity_and_merged_inference(bits):
    q, oq, x, xs, spec, cores, cores_np = _case(1024, 1024, 64, bits, 8, 31)
    base = L.QuantizedLinear("w.base", q)
    ad = L.TTLinear("w", base, spec, cores)
    wt = L.tt_materialize(spec, cores)
    assert O.rel_err(_np(wt), O.tt_full(cores_np)) <= TOL_F32
    merged = L.tt_merge(ad)
    assert O.rel_err(_np(merged), O.qa_merge(oq, cores_np)) <= TOL_F32
    with pytest.raises(qa.ModelError, match="already merged"):
        L.tt_merge(ad)
    with pytest.raises(qa.ModelError, match="inference-only"):
        ad.backward(x, torch.zeros(64, 1024, device="cuda"), {})
    y = ad.forward(x)  # dense bf16 GEMM on W'
    assert O.rel_err(_np(y), xs.astype(np.float64) @ O.qa_merge(oq, cores_np).T) <= TOL_BF16


@pytest.mark.parametrize("N,K,bits,r", [(320, 520, 8, 8), (320, 520, 4, 16), (1280, 264, 4, 8)])
def test_fused_merge_ragged_tiles(N, K, bits, r):
    """The fused merge kernel (k_merge_fast) off the bench shapes: LoRA with N = 320 (64-row tiles, md % 256 != 0),
    K = 520 / 264 (a partial last column tile), int4 packing with an odd number of column pairs per tile edge and
    rank 16 (4 columns per lane, 2-byte code words copied by lane pairs): fp32 and bf16 W' against the oracle's
    dequantise + W_t route (lowrank.py:249-257)."""
    spec = L.TTSpec.lora(N, K, r)
    q, oq, x, xs, spec, cores, cores_np = _case(N, K, 16, bits, r, 41, spec)
    want = O.qa_merge(oq, cores_np)
    for dt, tol in ((torch.float32, TOL_F32), (torch.bfloat16, 2.0 ** -8)):
        ad = L.TTLinear("w", L.QuantizedLinear("w.base", q), spec, [c.clone() for c in cores])
        got = L.tt_merge(ad, dtype=dt)
        assert got.dtype == dt and O.rel_err(_np(got), want) <= tol, (dt, O.rel_err(_np(got), want))


def test_edge_cases():
    q = qa.quantize_rows(O.seeded_random(256, 512, 3, std=0.02), 8)
    spec = L.TTSpec.for_shape(256, 512, 4)
    cores = [torch.randn(spec.core_shape(k), device="cuda") * 0.01 for k in range(spec.d)]
    # empty token batch
    y = L.linear_forward(q, (spec, cores), torch.zeros(0, 512, device="cuda", dtype=torch.bfloat16))
    assert y.shape == (0, 256)
    # single token, 3-D input shape preserved
    x = torch.randn(1, 1, 512, device="cuda", dtype=torch.bfloat16)
    y = L.linear_forward(q, (spec, cores), x)
    assert y.shape == (1, 1, 256)
    # constant token rows (scale 0) go through the offset path exactly
    xc = torch.full((3, 512), 0.75, device="cuda")
    out = L.linear_forward(q, None, xc, debug=True)
    oq = O.quantize_rows(O.seeded_random(256, 512, 3, std=0.02), 8)
    assert O.rel_err(_np(out["y_f32"]), O.qmatmul(oq, np.full((3, 512), 0.75))) <= TOL_F32
    # shape mismatch and bad cores raise the reference's exception classes
    with pytest.raises(qa.QuantError):
        L.linear_forward(q, None, torch.zeros(4, 100, device="cuda"))
    with pytest.raises(qa.ModelError):
        L.linear_forward(q, (spec, cores[:2]), x)


@pytest.mark.parametrize("xdtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("N,K,T,spec", [(512, 512, 97, None), (512, 256, 70, L.TTSpec.lora(512, 256, 8))])
def test_activation_codes_offset_and_tie_rows(N, K, T, spec, xdtype):
    # Rows whose offset dwarfs their range (|lo| / step >> 255: a fused v*inv - lo*inv would cancel),
    # rows on a coarse grid (many exact rounding ties), constant rows and a one-hot row: the int32
    # accumulators (which see every activation code) must still match the reference bit for bit.
    q, oq, x, xs, spec, cores, cores_np = _case(N, K, T, 8, 8, 61, spec, xdtype)
    g = torch.Generator().manual_seed(5)
    base = torch.randn(T, K, generator=g)
    rows = [
        1000.0 + base[0:16] * 0.5,  # offset rows
        -3000.0 + base[16:24] * 4.0,
        torch.round(base[24:48] * 8.0) / 8.0,  # coarse grid: frequent exact ties
        torch.round(base[48:56] * 2.0) * 0.25 + 7.0,
        torch.full((4, K), 2.5),  # constant rows (step 0)
        torch.zeros(4, K),
        base[64:],
    ]
    X = torch.cat(rows)[:T]
    X[60] = 0.0
    X[60, 7] = 1.0  # one-hot
    x = X.to(xdtype).cuda()
    xs = x.float().cpu().numpy()
    out = L.linear_forward(q, (spec, cores), x, debug=True)
    ref = O.qa_linear_forward(xs, oq, cores_np)
    acc = _np(out["acc"]).astype(np.int64)
    assert np.array_equal(acc, ref["acc"]), f"accumulators differ in rows {np.unique(np.argwhere(acc != ref['acc'])[:, 0])[:10]}"
    assert O.rel_err(_np(L.linear_forward(q, (spec, cores), x)), ref["y"]) <= TOL_BF16


def test_determinism():
    q, oq, x, xs, spec, cores, _ = _case(1024, 1024, 512, 8, 8, 41)
    dy = torch.randn(512, 1024, device="cuda", dtype=torch.bfloat16)
    a = L.linear_forward(q, (spec, cores), x)
    b = L.linear_forward(q, (spec, cores), x)
    assert torch.equal(a, b)
    dx1, g1 = L.linear_backward(q, (spec, cores), x, dy)
    dx2, g2 = L.linear_backward(q, (spec, cores), x, dy)
    assert torch.equal(dx1, dx2)
    assert all(torch.equal(u, v) for u, v in zip(g1, g2))


def test_full_size_properties():
    # config-2 shape (4096x4096, 16384 tokens): exact accumulators on sampled entries, sampled
    # tokens against the oracle, and linearity of the backward in dy.
    N = K = 4096
    T = 16384
    torch.manual_seed(3)
    W = (torch.randn(N, K, device="cuda") * 0.02)
    q = qa.quantize_rows(W, 8)
    spec = L.TTSpec.for_shape(N, K, 8)
    cores = [torch.randn(spec.core_shape(k), device="cuda") * 0.01 for k in range(spec.d)]
    x = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    out = L.linear_forward(q, (spec, cores), x, debug=True)
    qx = qa.quantize_rows(x, 8)
    rows = torch.randint(0, T, (64,), device="cuda")
    cx = qx.codes[rows].double()
    exact = (cx @ q.codes.double().t()).long()  # fp64 is exact below 2^53
    assert torch.equal(exact, out["acc"][rows].long())
    oq = O.quantize_rows(W.cpu().numpy(), 8)
    cores_np = [c.cpu().numpy() for c in cores]
    ref = O.qa_linear_forward(x[rows].float().cpu().numpy(), oq, cores_np)
    assert O.rel_err(_np(out["y_bf16"][rows]), ref["y"]) <= TOL_BF16
    dy1 = torch.randn(T, N, device="cuda").to(torch.bfloat16)
    dy2 = torch.randn(T, N, device="cuda").to(torch.bfloat16)
    dsum = (dy1.float() + dy2.float()).to(torch.bfloat16)
    a, ga = L.linear_backward(q, (spec, cores), x, dy1)
    b, gb = L.linear_backward(q, (spec, cores), x, dy2)
    c, gc = L.linear_backward(q, (spec, cores), x, dsum)
    assert O.rel_err(_np(c), _np(a) + _np(b)) <= 2 * TOL_BF16
    for u, v, w in zip(ga, gb, gc):
        assert O.rel_err(_np(w), _np(u) + _np(v)) <= 2 * TOL_BF16


@pytest.mark.parametrize("ns,K,T,r", [((512, 768, 1024), 1024, 200, 8), ((1024, 2048), 512, 77, 8),
                                      ((512, 256), 1024, 64, 16),
                                      # decode sizes: the members' prologue + matrix-vector passes, chained
                                      ((512, 768, 1024), 1024, 1, 8), ((1024, 2048), 512, 5, 8),
                                      ((4096, 4096, 4096), 4096, 8, 8)])
def test_shared_input_group_matches_members(ns, K, T, r):
    """qa_group_forward / qa_group_backward (one x pass per direction for q / k / v-style members,
    transformer.py:862-874 / 919-944) give each member exactly its single-linear results; r = 16
    exercises the member-by-member fallback."""
    x = torch.from_numpy(O.seeded_random(T, K, 41)).cuda().to(torch.bfloat16)
    members, ref_members = [], []
    for i, N in enumerate(ns):
        q = qa.quantize_rows(O.seeded_random(N, K, 50 + i, std=0.02), 8)
        spec = L.TTSpec.for_shape(N, K, r)
        cores = [torch.from_numpy(c).cuda() for c in O.tt_init_cores(O.TTShape(spec.m, spec.n, spec.ranks), 60 + i)]
        members.append(L.TTLinear(f"m{i}", L.QuantizedLinear(f"m{i}.base", q), spec, [c.clone() for c in cores]))
        ref_members.append(L.TTLinear(f"m{i}", L.QuantizedLinear(f"m{i}.base", q), spec, [c.clone() for c in cores]))
    dys = [torch.from_numpy(O.seeded_random(T, N, 70 + i)).cuda().to(torch.bfloat16) for i, N in enumerate(ns)]
    ys = L.group_forward(members, x)
    g_grads, r_grads = {}, {}
    dxs = L.group_backward(members, x, dys, g_grads)
    for i, m in enumerate(ref_members):
        y_ref = m.forward(x)
        assert torch.equal(ys[i], y_ref), i
        dx_ref = m.backward(x, dys[i], r_grads)
        assert torch.equal(dxs[i], dx_ref), i
    assert sorted(g_grads) == sorted(r_grads)
    for k in g_grads:
        assert torch.equal(g_grads[k], r_grads[k]), k


@pytest.mark.parametrize("N,K,bits,r,spec", [(1024, 512, 8, 8, None), (768, 1024, 4, 8, None),
                                             (512, 256, 8, 8, "lora"), (512, 512, 8, 8, "base"),
                                             (1024, 1024, 8, 8, "config1")])
def test_decode_sized_batches(N, K, bits, r, spec):
    """1..8 tokens (KV-cached decoding, transformer.py:1043-1080) run the dp4a matrix-vector pass
    (gemv.cu): exact int32 products and the GEMM's epilogue, so y matches the oracle and the tcgen05
    path on the same rows."""
    if spec == "lora":
        spec = L.TTSpec.lora(N, K, r)
    elif spec == "config1":
        spec = L.TTSpec.for_shape(N, K, r)
    q, oq, x, xs, spec_, cores, cores_np = _case(N, K, 9, bits, r, 61, None if spec in (None, "base") else spec)
    adapter = None if spec == "base" else (spec_, cores)
    big = L.linear_forward(q, adapter, x)  # 9 tokens: the tensor-core path
    for T in (1, 2, 3, 5, 8):
        y = L.linear_forward(q, adapter, x[:T])
        ref = O.qa_linear_forward(xs[:T], oq, cores_np if adapter is not None else None)
        assert O.rel_err(_np(y), ref["y"]) <= TOL_BF16, T
        assert O.rel_err(_np(y), _np(big[:T])) <= 2 ** -7, T
        y32 = L.linear_forward(q, adapter, x[:T].float())
        assert O.rel_err(_np(y32), ref["y"]) <= 1e-4, T


@pytest.mark.parametrize("bits", [8, 4])
def test_decode_sized_group_matches_members(bits):
    """A shared-input group at decode size (q / k / v of one decoder layer, transformer.py:862-874 with 1..8
    tokens; member i + 1's prologue chained behind member i's matrix-vector pass): each member's y equals its own
    single-linear decode pass bit for bit and the oracle to bf16, int8 and int4 bases."""
    K = 1024
    members, refs = [], []
    for i, N in enumerate((1024, 512, 512)):
        W = O.seeded_random(N, K, 80 + i, std=0.02)
        q, oq = qa.quantize_rows(W, bits), O.quantize_rows(W, bits)
        spec = L.TTSpec.for_shape(N, K, 8)
        cores_np = O.tt_init_cores(O.TTShape(spec.m, spec.n, spec.ranks), 90 + i, std=0.05)
        cores = [torch.from_numpy(c).cuda() for c in cores_np]
        members.append(L.TTLinear(f"m{i}", L.QuantizedLinear(f"m{i}.base", q), spec, cores))
        refs.append((oq, cores_np))
    xs = O.seeded_random(8, K, 99)
    x = torch.from_numpy(xs).cuda().to(torch.bfloat16)
    xs_b = _np(x).astype(np.float64)
    for T in (1, 3, 8):
        ys = L.group_forward(members, x[:T])
        for i, m in enumerate(members):
            assert torch.equal(ys[i], m.forward(x[:T])), (T, i)
            ref = O.qa_linear_forward(xs_b[:T], refs[i][0], refs[i][1])
            assert O.rel_err(_np(ys[i]), ref["y"]) <= TOL_BF16, (T, i)


def test_config1_mse_training_step_matches_oracle():
    """BASELINE config 1 end to end on the device: W 1024^2 ~N(0, 0.02) int8, x [4, 128, 1024] ~N(0, 1) fp32, the
    balanced (4,16,16)^2 rank-8 tensor adapter with cores ~N(0, 0.01), forward, MSE to a seeded N(0, 1) target
    (qa_mse: the loss and dL/dy), backward — loss, dy, dx and the core gradients against the oracle (SURVEY §8a A15:
    the reference's loss is cross-entropy, so the oracle restates MSE)."""
    from paper_2402_13533_b200 import glue

    W = O.seeded_random(1024, 1024, 1, std=0.02)
    X = O.seeded_random(512, 1024, 2).reshape(4, 128, 1024)
    target = O.seeded_random(512, 1024, 3).reshape(4, 128, 1024)
    spec = L.TTSpec.for_shape(1024, 1024, 8)
    assert spec.m == (4, 16, 16) and spec.n == (4, 16, 16)
    cores_np = O.tt_init_cores(O.TTShape(spec.m, spec.n, spec.ranks), 4, std=0.01)
    q, oq = qa.quantize_rows(W, 8), O.quantize_rows(W, 8)
    lin = L.TTLinear("w", L.QuantizedLinear("w.base", q), spec, [torch.from_numpy(c).cuda() for c in cores_np])
    x = torch.from_numpy(X).cuda()
    y = lin.forward(x)
    assert y.shape == (4, 128, 1024) and y.dtype == torch.float32
    loss, dy = glue.mse(y, torch.from_numpy(target).cuda())
    ref_y = O.qa_linear_forward(X.reshape(512, 1024), oq, cores_np)["y"]
    ref_loss = O.mse_loss(ref_y, target.reshape(512, 1024))
    ref_dy = O.mse_grad(ref_y, target.reshape(512, 1024))
    assert abs(float(loss) - ref_loss) <= 1e-5 * ref_loss
    assert O.rel_err(_np(dy).reshape(512, 1024), ref_dy) <= 1e-4
    grads = {}
    dx = lin.backward(x, dy, grads)
    ref = O.qa_linear_backward(X.reshape(512, 1024), ref_dy, oq, cores_np)
    e_dx = O.rel_err(_np(dx).reshape(512, 1024), ref["dx"])
    e_g = [O.rel_err(_np(grads[f"w.core{k}"]), ref["dcores"][k]) for k in range(3)]
    print(f"config 1 MSE step: loss {float(loss):.6f} ({ref_loss:.6f}), dx {e_dx:.2e}, grads " +
          " ".join(f"{e:.2e}" for e in e_g))
    assert e_dx <= 1e-4 and max(e_g) <= TOL_GRAD_GENERIC
