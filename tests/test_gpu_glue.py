"""Decoder glue kernels (csrc/glue.cu through the C ABI) against plain PyTorch float32 references of the same
ops (transformer.py:478-519, 569-588, 872-874).  bf16 outputs: |got - want| <= 1e-2 (|want| + rms(want));
float32 outputs (inv, per-row losses): 1e-5 relative."""

import pytest
import torch

import oracle as O
from paper_2402_13533_b200 import glue

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _err(got, want):
    return O.rel_err(got.detach().float().cpu().numpy(), want.detach().float().cpu().numpy())


def _bf(*shape, seed=0, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("rows,dim", [(37, 256), (64, 1024), (19, 4096), (11, 8192)])
def test_rmsnorm_forward_and_residual_add(rows, dim):
    a, b = _bf(rows, dim, seed=1), _bf(rows, dim, seed=2, scale=0.5)
    gain = torch.rand(dim, device="cuda") + 0.5
    y, inv = glue.rmsnorm(a, gain)
    af = a.float()
    inv_ref = torch.rsqrt(af.pow(2).mean(-1) + 1e-5)
    assert torch.allclose(inv, inv_ref, rtol=1e-5)
    assert _err(y, af * inv_ref[:, None] * gain) < TOL
    y2, inv2, s = glue.rmsnorm(a, gain, b=b)
    assert torch.equal(s, a + b)  # the residual stream is the bf16 sum
    sf = s.float()
    assert _err(y2, sf * torch.rsqrt(sf.pow(2).mean(-1, keepdim=True) + 1e-5) * gain) < TOL


@pytest.mark.parametrize("rows,dim,ndy,with_res", [(37, 256, 1, False), (29, 4096, 3, True), (13, 8192, 2, True),
                                                   (64, 2048, 2, False)])
def test_rmsnorm_backward(rows, dim, ndy, with_res):
    x = _bf(rows, dim, seed=3)
    gain = torch.rand(dim, device="cuda") + 0.5
    dys = [_bf(rows, dim, seed=10 + i) for i in range(ndy)]
    dres = _bf(rows, dim, seed=20) if with_res else None
    _, inv = glue.rmsnorm(x, gain)
    dx = glue.rmsnorm_backward(x, gain, inv, dys, dres=dres)
    xr = x.float().requires_grad_(True)
    y = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * gain
    dsum = dys[0]
    for d in dys[1:]:
        dsum = dsum + d  # bf16 sum, as stored between the group's dx and the norm's backward
    (want,) = torch.autograd.grad(y, xr, dsum.float())
    if dres is not None:
        want = want + dres.float()
    assert _err(dx, want) < TOL


@pytest.mark.parametrize("b,l,heads,d", [(2, 64, 2, 128), (1, 100, 4, 64), (3, 17, 8, 16)])
def test_rope_matches_reference_and_inverts(b, l, heads, d):
    D = heads * d
    q, k = _bf(b * l, D, seed=4), _bf(b * l, D, seed=5)
    half = d // 2
    freqs = 10000.0 ** (-2.0 * torch.arange(half, dtype=torch.float64) / d)
    ang = torch.arange(l, dtype=torch.float64)[:, None] * freqs[None, :]
    cos, sin = torch.cos(ang).float().cuda(), torch.sin(ang).float().cuda()

    def ref(x):
        xh = x.float().view(b, l, heads, half, 2)
        e, o = xh[..., 0], xh[..., 1]
        c, s = cos[None, :, None, :], sin[None, :, None, :]
        return torch.stack((e * c - o * s, e * s + o * c), -1).reshape(b * l, D)

    want_q, want_k = ref(q), ref(k)
    q0 = q.clone()
    glue.rope_(q, k, cos, sin, heads, l)
    assert _err(q, want_q) < TOL and _err(k, want_k) < TOL
    glue.rope_(q, None, cos, sin, heads, l, inverse=True)
    assert _err(q, q0) < TOL


def test_swiglu_forward_backward():
    up, gate, dact = _bf(300, 512, seed=6), _bf(300, 512, seed=7, scale=3.0), _bf(300, 512, seed=8)
    act = glue.swiglu(up, gate)
    u = up.float().requires_grad_(True)
    g = gate.float().requires_grad_(True)
    a = u * torch.nn.functional.silu(g)
    assert _err(act, a) < TOL
    du, dg = torch.autograd.grad(a, (u, g), dact.float())
    dup, dgate = glue.swiglu_backward(up, gate, dact)
    assert _err(dup, du) < TOL and _err(dgate, dg) < TOL


@pytest.mark.parametrize("rows,vocab,scale", [(5, 512, 1.0), (33, 32000, 4.0), (3, 8, 30.0)])
def test_cross_entropy(rows, vocab, scale):
    logits = _bf(rows, vocab, seed=9, scale=scale)
    g = torch.Generator(device="cuda").manual_seed(3)
    tgt = torch.randint(0, vocab, (rows,), generator=g, device="cuda")
    loss, dl = glue.cross_entropy(logits, tgt)
    lf = logits.float().requires_grad_(True)
    want = torch.nn.functional.cross_entropy(lf, tgt)
    (dwant,) = torch.autograd.grad(want, lf)
    assert float(loss) == pytest.approx(float(want), rel=1e-5, abs=1e-6)
    assert _err(dl, dwant) < TOL


def test_glue_rejects_bad_shapes():
    x = _bf(4, 300)
    with pytest.raises((RuntimeError, ValueError)):  # dim 300 is not 256 * 2^k: QA_ERR_UNSUPPORTED
        glue.rmsnorm(x, torch.ones(300, device="cuda"))
    with pytest.raises(ValueError):
        glue.rmsnorm(x.float(), torch.ones(300, device="cuda"))
