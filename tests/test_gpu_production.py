"""GPU parity of the PRODUCTION kernels at the benchmark's shapes (config 2: the Llama-2-7B linear set, int8,
TT rank 8, 16384 tokens; config 5: a 70B gate projection, int4) against the oracle.

Every forward / backward here runs the persistent tcgen05 kernels the bench times: many output tiles per CTA
pair (double-buffered TMEM phases, the in-TMEM y2 fold of tile i-1 inside tile i's k-loop, the TMA-store
epilogue), the grouped raster (down-projection dX and the 70B int4 forward use group_m = 8), the shared-input
group passes (q/k/v and up/gate) and the single-CTA persistent kernel with several tiles per CTA.  The debug
outputs (int32 accumulators, y1, y2) are probe outputs of those same kernels (gemm_tc.cu probe_*).

The oracle runs on sampled token rows (y, dx) — every operand of a sampled row is exact, so sampling loses
nothing — and on all tokens for the adapter-core gradients (the staged oracle is O(T·K·r)).

Tolerances, |got - want| <= tol (|want| + rms(want)) (oracle.rel_err):
  exact : int32 accumulators
  1e-5  : y1 (fp32 epilogue of exact integers)
  1e-4  : y2 (3-term bf16 split of Z1 and V, fp32 accumulation)
  1e-2  : bf16 outputs (y, dx; dx also carries deq(W) rounded to bf16) and the adapter-core gradients (bf16
          intermediates in the fused dy pass), the latter also <= 3e-3 Frobenius-relative
"""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2402_13533_b200 as qa
from paper_2402_13533_b200 import linear as L

pytestmark = pytest.mark.gpu

TOL_Y1 = 1e-5
TOL_Y2 = 1e-4
# adapter-core gradients of the fast TT family: the fused dy pass feeds Z2 / dZ2 / dZ1 to mma.sync as bf16
# operands (measured 4.2e-3..7.2e-3 max-normalised at these shapes), so the bf16 bar applies, plus an
# average-case (Frobenius-relative) bar that a lost hi/lo split term would break
TOL_GRAD = 1e-2
TOL_GRAD_RMS = 3e-3
TOL_BF16 = 1e-2
BF16_ULP = 2.0 ** -7  # one bf16 ulp relative to the value (8-bit significand)


def _np(t):
    t = t.detach()
    return (t.float() if t.dtype == torch.bfloat16 else t).cpu().numpy()


def _oq(q, rows=None):
    """OQuant over the device codes (rows subset optional); the codes themselves are pinned bit-exact
    against the oracle by test_gpu_quant.py and re-checked on sampled rows below."""
    codes, scale, offset = _np(q.codes), _np(q.scale), _np(q.offset)
    if rows is not None:
        codes, scale, offset = codes[rows], scale[rows], offset[rows]
    return O.OQuant(codes.shape[0], q.cols, q.bits, codes, scale, offset)


def _check_weight_rows(W, q, rows):
    ref = O.quantize_rows(_np(W[rows]), q.bits)
    assert _np(q.codes)[rows].tobytes() == ref.codes.tobytes()
    assert _np(q.scale)[rows].tobytes() == ref.scale.tobytes()


def _ref_forward_rows(xs_rows, q, cores_np, cols):
    """Oracle y1 / y2 / acc of the sampled tokens, restricted to output columns `cols`."""
    oq = _oq(q, cols)
    qx = O.quantize_rows(xs_rows, 8)
    acc = O.int32_accumulators(qx, oq)
    y1 = O.qmatmul(oq, O.dequantize_rows(qx))
    y2 = xs_rows.astype(np.float64) @ O.tt_rows(cores_np, cols).T if cores_np is not None else 0.0 * y1
    return acc, y1, y2


def _ref_dx_rows(dys_rows, q, cores_np, chunk=2048):
    """dy·deq(W) + dy·W_t for the sampled tokens, over chunks of weight rows (the 70B grid is 1.9 GB in fp64)."""
    out = np.zeros((dys_rows.shape[0], q.cols))
    for n0 in range(0, q.rows, chunk):
        rows = np.arange(n0, min(q.rows, n0 + chunk))
        d = dys_rows[:, rows].astype(np.float64)
        out += O.qmatmul_t(_oq(q, rows), d)
        if cores_np is not None:
            out += d @ O.tt_rows(cores_np, rows)
    return out


def _member(N, K, bits, r, seed, std=0.01, device_w=False):
    if device_w:
        g = torch.Generator(device="cuda").manual_seed(seed)
        W = torch.randn(N, K, generator=g, device="cuda") * 0.02
    else:
        W = torch.from_numpy(O.seeded_random(N, K, seed, std=0.02)).cuda()
    q = qa.quantize_rows(W, bits)
    spec = L.TTSpec.for_shape(N, K, r)
    cores_np = O.tt_init_cores(O.TTShape(spec.m, spec.n, spec.ranks), seed + 1, std=std)
    lin = L.TTLinear(f"m{seed}", L.QuantizedLinear(f"m{seed}.base", q), spec,
                     [torch.from_numpy(c).cuda() for c in cores_np])
    return W, q, spec, cores_np, lin


def _tokens(T, K, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(T, K, generator=g, device="cuda").to(torch.bfloat16)
    return x


def _probe_check(lin, cores_np, x, rows, cols, y_prod):
    """Probe run of the production GEMM: exact accumulators, y1, y2, y; and the production y (TMA-store
    epilogue, y2 folded in TMEM) within one bf16 ulp of the probe's y."""
    out = L.linear_forward(lin.base.q, (lin.spec, lin._core_tensors()), x, debug=True)
    xs = _np(x[rows])
    acc, y1, y2 = _ref_forward_rows(xs, lin.base.q, cores_np, cols)
    rt = torch.from_numpy(rows).cuda()
    ct = torch.from_numpy(cols).cuda()
    got_acc = _np(out["acc"][rt][:, ct]).astype(np.int64)
    assert np.array_equal(got_acc, acc), np.argwhere(got_acc != acc)[:5]
    g_y2 = _np(out["y2"][rt][:, ct])
    g_y1 = _np(out["y_f32"][rt][:, ct]) - g_y2
    e1, e2 = O.rel_err(g_y1, y1), O.rel_err(g_y2, y2)
    ey = O.rel_err(_np(out["y_bf16"][rt][:, ct]), y1 + y2)
    print(f"probe {lin.base.q.rows}x{lin.base.q.cols} T={x.shape[0]}: y1 {e1:.2e} y2 {e2:.2e} y {ey:.2e}")
    assert e1 <= TOL_Y1 and e2 <= TOL_Y2 and ey <= TOL_BF16, (e1, e2, ey)
    eprod = O.rel_err(_np(y_prod), _np(out["y_bf16"]))
    assert eprod <= BF16_ULP, eprod
    return float(np.sqrt(np.mean(y2 ** 2)) / np.sqrt(np.mean((y1 + y2) ** 2)))


def _grads_check(members, cores_list, x, dys, grads):
    xs = _np(x)
    for m, cn, dy in zip(members, cores_list, dys):
        _, ref = O.tt_backward_staged(xs, _np(dy), cn)
        for k, p in enumerate(m.cores):
            e, f = O.rel_err(_np(grads[p.name]), ref[k]), O.rel_rms(_np(grads[p.name]), ref[k])
            print(f"  {p.name} grad err {e:.2e} rms {f:.2e}")
            assert e <= TOL_GRAD and f <= TOL_GRAD_RMS, (p.name, e, f)


def _dx_check(members, cores_list, dys, dxs, rows):
    for m, cn, dy, dx in zip(members, cores_list, dys, dxs):
        want = _ref_dx_rows(_np(dy[torch.from_numpy(rows).cuda()]), m.base.q, cn)
        e = O.rel_err(_np(dx[torch.from_numpy(rows).cuda()]), want)
        print(f"  {m.name} dx err {e:.2e}")
        assert e <= TOL_BF16, (m.name, e)


T_BENCH = 16384


def _sample(T, n, seed):
    rng = np.random.default_rng(seed)
    # first and last tiles, the pair boundary (row 128) and random rows
    return np.unique(np.concatenate([[0, 127, 128, 255, 256, T - 1], rng.integers(0, T, n)]))


def test_qkv_group_bench_step_matches_oracle():
    """The bench's q/k/v step: qa_group_forward + qa_group_backward over 3 x 4096^2 int8, T = 16384."""
    T, K = T_BENCH, 4096
    parts = [_member(4096, K, 8, 8, 100 + 10 * i) for i in range(3)]
    members = [p[4] for p in parts]
    cores_list = [p[3] for p in parts]
    _check_weight_rows(parts[0][0], parts[0][1], np.array([0, 1, 4095]))
    x = _tokens(T, K, 7)
    rows = _sample(T, 40, 1)
    cols = np.arange(K)
    ys = L.group_forward(members, x)
    # production outputs of every member against the oracle on the sampled tokens
    xs = _np(x[torch.from_numpy(rows).cuda()])
    for m, cn, y in zip(members, cores_list, ys):
        acc, y1, y2 = _ref_forward_rows(xs, m.base.q, cn, cols)
        e = O.rel_err(_np(y[torch.from_numpy(rows).cuda()]), y1 + y2)
        print(f"  {m.name} y err {e:.2e}")
        assert e <= TOL_BF16, e
    _probe_check(members[0], cores_list[0], x, rows, cols, ys[0])
    dys = [_tokens(T, 4096, 20 + i) for i in range(3)]
    grads = {}
    dxs = L.group_backward(members, x, dys, grads)
    _dx_check(members, cores_list, dys, dxs, rows)
    _grads_check(members, cores_list, x, dys, grads)


def test_up_gate_group_and_down_bench_step_match_oracle():
    """The bench's MLP step: up/gate (2 x 11008x4096) as a shared-input group and down (4096x11008), T = 16384.
    The down projection's dX GEMM runs the grouped raster (group_m = 8)."""
    T = T_BENCH
    parts = [_member(11008, 4096, 8, 8, 200 + 10 * i) for i in range(2)]
    members = [p[4] for p in parts]
    cores_list = [p[3] for p in parts]
    x = _tokens(T, 4096, 8)
    rows = _sample(T, 24, 2)
    cols = np.arange(0, 11008, 3)
    ys = L.group_forward(members, x)
    xs = _np(x[torch.from_numpy(rows).cuda()])
    for m, cn, y in zip(members, cores_list, ys):
        _, y1, y2 = _ref_forward_rows(xs, m.base.q, cn, cols)
        e = O.rel_err(_np(y[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()]), y1 + y2)
        assert e <= TOL_BF16, e
    dys = [_tokens(T, 11008, 30 + i) for i in range(2)]
    grads = {}
    dxs = L.group_backward(members, x, dys, grads)
    _dx_check(members, cores_list, dys, dxs, rows)
    _grads_check(members, cores_list, x, dys, grads)
    # down projection: single linear through the recompute window (forward_save -> backward_saved)
    Wd, qd, specd, cnd, down = _member(4096, 11008, 8, 8, 300)
    h = _tokens(T, 11008, 9)
    yd = down.forward(h)
    _probe_check(down, cnd, h, rows, np.arange(4096), yd)
    dyd = _tokens(T, 4096, 40)
    gd = {}
    dxd = down.backward(h, dyd, gd)
    _dx_check([down], [cnd], [dyd], [dxd], rows)
    _grads_check([down], [cnd], h, [dyd], gd)


def test_y2_visible_at_bench_shape():
    """Cores with std 0.1 make y2 about half of y, so the bf16 check on y sees the in-TMEM fold directly."""
    W, q, spec, cores_np, lin = _member(4096, 4096, 8, 8, 400, std=0.1)
    x = _tokens(T_BENCH, 4096, 10)
    y = lin.forward(x)  # qa_linear_forward_save: the recompute-window forward of the bench's o projection
    rows = _sample(T_BENCH, 40, 3)
    share = _probe_check(lin, cores_np, x, rows, np.arange(4096), y)
    assert share > 0.2, share
    _, y1, y2 = _ref_forward_rows(_np(x[torch.from_numpy(rows).cuda()]), q, cores_np, np.arange(4096))
    assert O.rel_err(_np(y[torch.from_numpy(rows).cuda()]), y1 + y2) <= TOL_BF16
    # dropping y2 must fail this bar by a wide margin (the check is not blind to the adapter)
    assert O.rel_err(y1, y1 + y2) > 10 * TOL_BF16


def test_int4_70b_gate_grouped_raster_matches_oracle():
    """Config 5's gate projection (28672 x 8192, int4, r = 8) at 4096 tokens: the int8 forward runs the
    grouped raster (group_m = 8) over 16 M-tiles x 112 N-tiles, several tiles per CTA pair."""
    T = 4096
    W, q, spec, cores_np, lin = _member(28672, 8192, 4, 8, 500, device_w=True)
    _check_weight_rows(W, q, np.array([0, 5, 28671]))
    x = _tokens(T, 8192, 11)
    y = lin.forward(x)
    rows = _sample(T, 16, 4)
    cols = np.unique(np.concatenate([np.arange(0, 28672, 97), [0, 255, 256, 28671]]))
    _probe_check(lin, cores_np, x, rows, cols, y)
    dy = _tokens(T, 28672, 41)
    grads = {}
    dx = lin.backward(x, dy, grads)
    _dx_check([lin], [cores_np], [dy], [dx], rows[:6])
    _grads_check([lin], [cores_np], x, [dy], grads)


def test_single_cta_persistent_kernel_multi_tile():
    """M <= 128 runs k_gemm_tc_p; N = 49152 gives 192 output tiles over 148 CTAs (two tiles on some)."""
    T, N, K = 100, 49152, 256
    W, q, spec, cores_np, lin = _member(N, K, 8, 8, 600)
    x = _tokens(T, K, 12)
    y = lin.forward(x)
    rows = np.arange(T)
    cols = np.arange(N)
    _probe_check(lin, cores_np, x, rows, cols, y)
    dy = _tokens(T, N, 42)
    grads = {}
    dx = lin.backward(x, dy, grads)
    _dx_check([lin], [cores_np], [dy], [dx], rows)
    _grads_check([lin], [cores_np], x, [dy], grads)


@pytest.mark.parametrize("shape", [(28672, 8192, 4), (1024, 8192, 4), (4096, 11008, 8)])
@pytest.mark.parametrize("kind", ["tt", "lora"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_merge_matches_oracle_at_benchmark_shapes(shape, kind, dtype):
    """qa_merge as the bench times it (config 5's 70B gate and GQA k/v shapes, int4; the 7B down projection,
    int8): the fused fast-family merge (prefix contraction in registers) for the pinned TT modes and LoRA,
    against dequantize_rows + W_t (lowrank.py:245-257 via :249-252) on sampled rows.  fp32 output within 1e-5,
    bf16 output within one bf16 ulp."""
    N, K, bits = shape
    g = torch.Generator(device="cuda").manual_seed(N + K)
    q = qa.quantize_rows(torch.randn(N, K, generator=g, device="cuda") * 0.02, bits)
    spec = L.TTSpec.for_shape(N, K, 8) if kind == "tt" else L.TTSpec.lora(N, K, 8)
    cores_np = O.tt_init_cores(O.TTShape(spec.m, spec.n, spec.ranks), 7, std=0.05)
    lin = L.TTLinear("w", L.QuantizedLinear("w.base", q), spec, [torch.from_numpy(c).cuda() for c in cores_np])
    merged = L.tt_merge(lin, dtype)
    rows = _sample(N, 24, 5)
    want = O.dequantize_rows(_oq(q, rows)) + O.tt_rows(cores_np, rows)
    got = _np(merged[torch.from_numpy(rows).cuda()])
    e = O.rel_err(got, want)
    print(f"merge {kind} {N}x{K} int{bits} {dtype}: {e:.2e}")
    assert e <= (1e-5 if dtype == torch.float32 else BF16_ULP / 2), e
    # W_t alone (qa_tt_materialize, same fused kernel without codes)
    wt = L.tt_materialize(spec, lin._core_tensors())
    assert O.rel_err(_np(wt[torch.from_numpy(rows).cuda()]), O.tt_rows(cores_np, rows)) <= 1e-5


@pytest.mark.parametrize("T", [1, 8])
def test_decode_at_benchmark_shapes(T):
    """The decode step the bench times (KV-cached decoding, transformer.py:1043-1080) at the 7B shapes: the
    up / gate group (one prologue launch for both members, one matrix-vector launch over their 22016 rows, each
    warp holding a 4096-column slice in registers) and the down projection (K = 11008: three register rounds per
    warp), against the oracle on all tokens and sampled output columns (y within the bf16 bar)."""
    rng = np.random.default_rng(5)
    up = _member(11008, 4096, 8, 8, 301, std=0.05, device_w=True)
    gate = _member(11008, 4096, 8, 8, 303, std=0.05, device_w=True)
    down = _member(4096, 11008, 8, 8, 305, std=0.05, device_w=True)
    x = _tokens(T, 4096, 307)
    xd = _tokens(T, 11008, 309)
    ys = L.group_forward([up[4], gate[4]], x)
    yd = down[4].forward(xd)
    for (W, q, spec, cores_np, lin), y, xin in ((up, ys[0], x), (gate, ys[1], x), (down, yd, xd)):
        cols = np.sort(rng.choice(q.rows, 512, replace=False))
        _check_weight_rows(W, q, cols[:64])
        _, y1, y2 = _ref_forward_rows(_np(xin), q, cores_np, cols)
        e = O.rel_err(_np(y[:, torch.from_numpy(cols).cuda()]), y1 + y2)
        print(f"decode {q.rows}x{q.cols} T={T}: y err {e:.2e}")
        assert e <= TOL_BF16, e
        # bit-identical to the single-linear decode pass
        assert torch.equal(y, lin.forward(xin))
