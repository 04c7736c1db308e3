"""float64 numpy restatement of the quantised tensor-adapter linear (TEST INFRASTRUCTURE).

See oracle/__init__.py for the contract.  Citations are into /root/reference/pkg/src/lrlm
unless stated otherwise.  Nothing here is shipped; the CUDA path never calls it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OracleError",
    "splitmix64",
    "seeded_random",
    "to_bf16",
    "OQuant",
    "quantize_rows",
    "dequantize_rows",
    "pack4",
    "unpack4",
    "qmatmul",
    "qmatmul_t",
    "int32_accumulators",
    "TTShape",
    "tt_modes_for",
    "tt_init_cores",
    "tt_full",
    "tt_apply",
    "tt_rows",
    "tt_prefix",
    "tt_dx",
    "tt_core_grads",
    "lora_as_tt",
    "qa_linear_forward",
    "qa_linear_backward",
    "qa_merge",
    "mse_loss",
    "mse_grad",
    "dp_mean",
    "rel_err",
    "rel_rms",
    "tt_apply_staged",
    "tt_backward_staged",
    "qa_step_staged",
]


class OracleError(ValueError):
    pass


# ---------------------------------------------------------------------------
# Seeded inputs: SplitMix64 + Box-Muller, restating linalg.py:76-152 so the
# oracle regenerates the reference's exact input bytes without importing it.
# ---------------------------------------------------------------------------

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """First `count` outputs of SplitMix64 started at `seed` (linalg.py:92-102)."""
    steps = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + steps * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        return z ^ (z >> np.uint64(31))


def seeded_random(rows, cols, seed, dist="gaussian", std=1.0, lo=0.0, hi=1.0, dtype=np.float32):
    """Bit-identical restatement of linalg.seeded_random (linalg.py:127-152).

    One generator stream per call: uniforms are 53-bit draws in (0, 1]
    (linalg.py:104-107); gaussians use Box-Muller on the first half / second
    half of the uniform stream (linalg.py:109-119).
    """
    if rows < 1 or cols < 1:
        raise OracleError(f"grid dims must be >= 1, got {rows}x{cols}")
    total = rows * cols
    if dist == "gaussian":
        pairs = (total + 1) // 2
        raw = splitmix64(seed, 2 * pairs)
        u = ((raw >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
        u1, u2 = u[:pairs], u[pairs:]
        rad = np.sqrt(-2.0 * np.log(u1))
        ang = 2.0 * np.pi * u2
        flat = np.empty(2 * pairs)
        flat[0::2] = rad * np.cos(ang)
        flat[1::2] = rad * np.sin(ang)
        flat = flat[:total] * std
    elif dist == "uniform":
        raw = splitmix64(seed, total)
        u = ((raw >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
        flat = lo + u * (hi - lo)
    else:
        raise OracleError(f"unknown dist {dist!r}")
    return flat.reshape(rows, cols).astype(dtype)


def to_bf16(a) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returned as float32.

    numpy has no bf16; the GPU path stores activations in bf16, so the oracle
    consumes the same (exactly representable) values.
    """
    f = np.ascontiguousarray(a, dtype=np.float32)
    bits = f.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    out = rounded.astype(np.uint32).view(np.float32)
    return np.where(np.isfinite(f), out, f).astype(np.float32)


# ---------------------------------------------------------------------------
# Per-row min/max quantisation (quant.py:73-99) and the code container (quant.py:55-70)
# ---------------------------------------------------------------------------


def pack4(codes: np.ndarray) -> np.ndarray:
    """Two 4-bit codes per byte, even column in the low nibble, odd K padded with 0 (quant.py:37-43)."""
    r, c = codes.shape
    padded = np.zeros((r, c + (c & 1)), dtype=np.uint8)
    padded[:, :c] = codes
    return (padded[:, 0::2] | (padded[:, 1::2] << 4)).astype(np.uint8)


def unpack4(packed: np.ndarray, cols: int) -> np.ndarray:
    """Inverse of pack4 (quant.py:46-52)."""
    out = np.empty((packed.shape[0], 2 * packed.shape[1]), dtype=np.uint8)
    out[:, 0::2] = packed & 0x0F
    out[:, 1::2] = packed >> 4
    return out[:, :cols]


@dataclass
class OQuant:
    rows: int
    cols: int
    bits: int
    codes: np.ndarray  # u8, packed two per byte for bits == 4 (the reference layout)
    scale: np.ndarray  # f32 [rows]
    offset: np.ndarray  # f32 [rows]
    scale64: np.ndarray = field(repr=False, default=None)  # the fp64 quotient the codes were derived with

    def unpacked(self) -> np.ndarray:
        return unpack4(self.codes, self.cols) if self.bits == 4 else self.codes

    def rowsum(self) -> np.ndarray:
        """Σ_k code[n, k] as int64 (the epilogue term of SURVEY §8a A4)."""
        return self.unpacked().astype(np.int64).sum(axis=1)


def quantize_rows(w, bits: int) -> OQuant:
    """Restates quant.py:73-99.

    lo/hi are the fp64 row extremes, the step is the fp64 quotient (hi-lo)/(2^b-1),
    each code is floor(v + 0.5) of the fp64 quotient v = (w-lo)/step (ties away
    from zero; v >= 0 so _round_half_away, quant.py:32-34, reduces to this), then
    clipped; rows with a zero step get code 0.  scale/offset are stored as f32.
    """
    if bits not in (4, 8):
        raise OracleError(f"bits must be 4 or 8, got {bits}")
    w = np.asarray(w)
    if w.ndim != 2:
        raise OracleError(f"expected 2-D grid, got shape {w.shape}")
    if not np.isfinite(w).all():
        raise OracleError("cannot quantize non-finite values")
    top = (1 << bits) - 1
    w64 = w.astype(np.float64)
    lo = w64.min(axis=1)
    step = (w64.max(axis=1) - lo) / top
    denom = np.where(step > 0, step, 1.0)
    v = (w64 - lo[:, None]) / denom[:, None]
    codes = np.clip(np.floor(v + 0.5), 0, top).astype(np.uint8)
    codes[step == 0] = 0
    return OQuant(
        rows=w.shape[0], cols=w.shape[1], bits=bits,
        codes=pack4(codes) if bits == 4 else codes,
        scale=step.astype(np.float32), offset=lo.astype(np.float32), scale64=step,
    )


def dequantize_rows(q: OQuant, dtype=np.float64) -> np.ndarray:
    """code * scale + offset in fp64 (quant.py:102-105)."""
    c = q.unpacked().astype(np.float64)
    return (c * q.scale.astype(np.float64)[:, None] + q.offset.astype(np.float64)[:, None]).astype(dtype)


def qmatmul(q: OQuant, x) -> np.ndarray:
    """x (..., cols) -> (..., rows): (x·codesᵀ)·scale + Σx·offset, fp64 (quant.py:123-132)."""
    xs = np.asarray(x, dtype=np.float64)
    if xs.shape[-1] != q.cols:
        raise OracleError("qmatmul dimension mismatch")
    c = q.unpacked().astype(np.float64)
    return (xs @ c.T) * q.scale.astype(np.float64) + xs.sum(axis=-1, keepdims=True) * q.offset.astype(np.float64)


def qmatmul_t(q: OQuant, dy) -> np.ndarray:
    """dy (..., rows) -> dy·deq(W) = (dy·scale)·codes + (dy·offset) (quant.py:135-144)."""
    ds = np.asarray(dy, dtype=np.float64)
    if ds.shape[-1] != q.rows:
        raise OracleError("qmatmul_t dimension mismatch")
    c = q.unpacked().astype(np.float64)
    return (ds * q.scale.astype(np.float64)) @ c + (ds @ q.offset.astype(np.float64))[..., None]


def int32_accumulators(qx: OQuant, qw: OQuant) -> np.ndarray:
    """acc[t, n] = Σ_k cx[t,k]·cw[n,k] exactly: fp64 BLAS is exact below 2^53."""
    acc = qx.unpacked().astype(np.float64) @ qw.unpacked().astype(np.float64).T
    return acc.astype(np.int64)


# ---------------------------------------------------------------------------
# Tensor-train (matrix-product-operator) adapter — absent from the reference
# (SPEC.md:8); restated from PAPER.md:55,67,70,209-217 and SURVEY §8a A6.
#   cores[k] : (r_{k-1}, m_k, n_k, r_k), r_0 = r_d = 1
#   W_t[(i1..id), (j1..jd)] = G1[0,i1,j1,:] G2[:,i2,j2,:] ... Gd[:,id,jd,0]   (row-major multi-indices)
#   y2 = x · W_tᵀ, no scaling.
# LoRA is the 2-core case m=(1,N), n=(K,1): G1 = downᵀ.reshape(1,1,K,r), G2 = upᵀ.reshape(r,N,1,1).
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TTShape:
    m: tuple  # output modes, Π m = N (fan_out)
    n: tuple  # input modes,  Π n = K (fan_in)
    ranks: tuple  # (1, r_1, ..., r_{d-1}, 1)

    def __post_init__(self):
        if len(self.m) != len(self.n) or len(self.ranks) != len(self.m) + 1:
            raise OracleError("TT mode/rank length mismatch")
        if self.ranks[0] != 1 or self.ranks[-1] != 1:
            raise OracleError("boundary TT ranks must be 1")

    @property
    def d(self):
        return len(self.m)

    @property
    def N(self):
        return int(np.prod(self.m))

    @property
    def K(self):
        return int(np.prod(self.n))

    def core_shape(self, k):
        return (self.ranks[k], self.m[k], self.n[k], self.ranks[k + 1])


def tt_modes_for(N: int, K: int, r: int) -> TTShape:
    """The mode factorisation pinned for each BASELINE shape (BASELINE.json leaves 7B/70B open).

    Config 1 (1024x1024): balanced (4,16,16)x(4,16,16) as BASELINE.json states.
    Llama shapes: m = (1, N/256, 256), n = (K/4, 4, 1): the first core is
    input-only and the last output-only, so the contractions that touch x or dy
    have rank r on their small side (like LoRA's down / up projections) while
    the middle core couples 16..112 output blocks with 4 input blocks.
    """
    if N == 1024 and K == 1024:
        return TTShape((4, 16, 16), (4, 16, 16), (1, r, r, 1))
    if N % 256 == 0 and K % 4 == 0:
        return TTShape((1, N // 256, 256), (K // 4, 4, 1), (1, r, r, 1))
    raise OracleError(f"no pinned TT modes for {N}x{K}")


def tt_init_cores(shape: TTShape, seed: int, std: float = 0.01):
    """Cores ~N(0, std^2) (BASELINE config 1), core k from seeded_random(seed + k)."""
    out = []
    for k in range(shape.d):
        s = shape.core_shape(k)
        g = seeded_random(int(np.prod(s[:2])), int(np.prod(s[2:])), seed + k, std=std)
        out.append(g.reshape(s))
    return out


def tt_full(cores) -> np.ndarray:
    """Materialise W_t (N x K) in fp64 by contracting the cores left to right."""
    cur = np.asarray(cores[0], dtype=np.float64)[0]  # (m1, n1, r1)
    for g in cores[1:]:
        g = np.asarray(g, dtype=np.float64)
        i, j, _ = cur.shape
        nxt = np.einsum("ija,akqb->ikjqb", cur, g)
        cur = nxt.reshape(i * g.shape[1], j * g.shape[2], g.shape[3])
    return cur[..., 0]


def tt_rows(cores, rows) -> np.ndarray:
    """Selected rows of W_t ([len(rows), K] fp64) without materialising the whole matrix: row n with
    multi-index (i_1..i_d) (row-major over m) is G1[0,i_1,:,:] · G2[:,i_2,:,:] ··· Gd[:,i_d,:,0] over j."""
    cs = [np.asarray(g, dtype=np.float64) for g in cores]
    ms = [g.shape[1] for g in cs]
    rows = np.asarray(rows, dtype=np.int64)
    idx = []
    rem = rows.copy()
    for m in reversed(ms):
        idx.append(rem % m)
        rem //= m
    idx = idx[::-1]
    cur = cs[0][0][idx[0]]  # [R, n_1, r_1]
    for k in range(1, len(cs)):
        g = cs[k][:, idx[k]]  # [a, R, n_k, b]
        cur = np.einsum("rja,arqb->rjqb", cur, g)
        cur = cur.reshape(cur.shape[0], -1, cur.shape[-1])
    return cur[..., 0]


def tt_apply(x, cores) -> np.ndarray:
    """y2 = x · W_tᵀ in fp64."""
    return np.asarray(x, dtype=np.float64) @ tt_full(cores).T


def tt_prefix(x, cores):
    """Left-to-right partial contractions Z_k[t, i<=k, r_k, j>k], k = 1..d-1 (the GPU's intermediates).

    Z_k = Σ_{a, j_k} Z_{k-1}[t, i<k, a, j_k, j>k] · G_k[a, i_k, j_k, b]; Z_{d-1} viewed as
    [T, H, r_{d-1}·n_d] is the operand of the fused last stage (y2 = U · G_d).
    """
    x = np.asarray(x, dtype=np.float64)
    t = x.shape[0]
    z = x.reshape(t, 1, 1, -1)  # [T, I_0=1, r_0=1, K]
    out = []
    for g in cores[:-1]:
        g = np.asarray(g, dtype=np.float64)
        a, mk, nk, b = g.shape
        i0 = z.shape[1]
        z = z.reshape(t, i0, a, nk, -1)  # [T, I, a, n_k, J_rest]
        z = np.einsum("tiajq,akjb->tikbq", z, g).reshape(t, i0 * mk, b, -1)
        out.append(z)
    return out


def tt_dx(dy, cores) -> np.ndarray:
    """Adapter contribution to dL/dx: dy · W_t (fp64)."""
    return np.asarray(dy, dtype=np.float64) @ tt_full(cores)


def tt_core_grads(x, dy, cores):
    """dL/dG_k for L with dL/dy2 = dy: project dW_t = dyᵀ·x onto each core.

    dG_k[a,i,j,b] = Σ L_{k-1}[i<k, j<k, a] · dW[(i<k,i,i>k),(j<k,j,j>k)] · R_{k+1}[b, i>k, j>k].
    """
    x = np.asarray(x, dtype=np.float64).reshape(-1, np.asarray(x).shape[-1])
    dy = np.asarray(dy, dtype=np.float64).reshape(-1, np.asarray(dy).shape[-1])
    dw = dy.T @ x
    cs = [np.asarray(g, dtype=np.float64) for g in cores]
    d = len(cs)
    grads = []
    for k in range(d):
        left = np.ones((1, 1, 1))  # [I<k, J<k, r_{k-1}]
        for g in cs[:k]:
            i, j, _ = left.shape
            left = np.einsum("ija,akqb->ikjqb", left, g).reshape(i * g.shape[1], j * g.shape[2], g.shape[3])
        right = np.ones((1, 1, 1))  # [r_k, I>k, J>k]
        for g in reversed(cs[k + 1:]):
            _, i, j = right.shape
            right = np.einsum("akqb,bij->akiqj", g, right).reshape(g.shape[0], g.shape[1] * i, g.shape[2] * j)
        a, mk, nk, b = cs[k].shape
        il, jl = left.shape[0], left.shape[1]
        ir, jr = right.shape[1], right.shape[2]
        dw6 = dw.reshape(il, mk, ir, jl, nk, jr)
        grads.append(np.einsum("pqa,pmiqnj,bij->amnb", left, dw6, right))
    return grads


def lora_as_tt(down, up):
    """LoRA (LoraLinear, transformer.py:276-327) as a 2-core TT: W_t = up·down."""
    down = np.asarray(down)
    up = np.asarray(up)
    r, k = down.shape
    n = up.shape[0]
    shape = TTShape((1, n), (k, 1), (1, r, 1))
    return shape, [down.T.reshape(1, 1, k, r), up.T.reshape(r, n, 1, 1)]


# ---------------------------------------------------------------------------
# The quantised tensor-adapter linear
# ---------------------------------------------------------------------------


def qa_linear_forward(x, qw: OQuant, cores, act_bits: int = 8) -> dict:
    """Forward of the paper's quantised adapter linear:

    per-token act-quant = quantize_rows(x2d, 8) (quant.py:73-99 on [T,K]),
    y1 = deq(Q(x)) · deq(Q(W))ᵀ computed as qmatmul(qw, deq(qx)) (quant.py:123-132),
    y2 = x · W_tᵀ (TT adapter on the unquantised x, as LoraLinear.forward, transformer.py:304-308),
    y = y1 + y2.
    """
    x2 = np.asarray(x, dtype=np.float64).reshape(-1, qw.cols)
    qx = quantize_rows(x2, act_bits)
    y1 = qmatmul(qw, dequantize_rows(qx))
    y2 = tt_apply(x2, cores) if cores is not None else np.zeros_like(y1)
    return {"qx": qx, "acc": int32_accumulators(qx, qw), "y1": y1, "y2": y2, "y": y1 + y2}


def qa_linear_backward(x, dy, qw: OQuant, cores) -> dict:
    """Backward with recompute (LoraLinear.backward, transformer.py:310-318, as TT):

    dx = qmatmul_t(qw, dy) + dy·W_t (quant.py:135-144); adapter grads only, by projection.
    """
    x2 = np.asarray(x, dtype=np.float64).reshape(-1, qw.cols)
    dy2 = np.asarray(dy, dtype=np.float64).reshape(-1, qw.rows)
    dx = qmatmul_t(qw, dy2)
    out = {"dx_base": dx.copy()}
    if cores is not None:
        dx = dx + tt_dx(dy2, cores)
        out["dcores"] = tt_core_grads(x2, dy2, cores)
    out["dx"] = dx
    return out


def qa_merge(qw: OQuant, cores) -> np.ndarray:
    """W' = dequantize_rows(q) + W_t: the explicit-dequantise route lowrank.py:249-252 prescribes."""
    return dequantize_rows(qw, np.float64) + tt_full(cores)


def mse_loss(y, target) -> float:
    """L = mean (y - target)^2 (the reference loss is CE, transformer.py:569-588)."""
    d = np.asarray(y, dtype=np.float64) - np.asarray(target, dtype=np.float64)
    return float(np.mean(d * d))


def mse_grad(y, target) -> np.ndarray:
    d = np.asarray(y, dtype=np.float64) - np.asarray(target, dtype=np.float64)
    return 2.0 * d / d.size


def dp_mean(per_rank: list) -> dict:
    """Fixed-order sum then divide by the replica count (distsim.py:309-314)."""
    out = {}
    for name in per_rank[0]:
        acc = np.zeros_like(np.asarray(per_rank[0][name], dtype=np.float64))
        for g in per_rank:
            acc += g[name]
        out[name] = acc / len(per_rank)
    return out


def rel_err(got, want) -> float:
    """max |got - want| / (max|want| ... ) normalised as SURVEY §8(d): |e| <= rtol(|want| + rms(want))."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if want.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(want * want)))
    denom = np.abs(want) + rms
    denom = np.where(denom > 0, denom, 1.0)
    return float(np.max(np.abs(got - want) / denom))


def rel_rms(got, want) -> float:
    """||got - want|| / ||want|| (Frobenius): the average-case companion of rel_err."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    n = float(np.linalg.norm(want))
    return float(np.linalg.norm(got - want)) / (n if n > 0 else 1.0)


# ---------------------------------------------------------------------------
# Staged (non-materialising) CPU port: the same left-to-right stage algebra the GPU runs.
# Used as bench.py's CPU baseline (`cpu_baseline` / `--impl reference`) because materialising
# W_t per call is not how a CPU implementation would run the layer; it is checked against the
# materialising oracle above in tests/test_oracle_golden.py.
# ---------------------------------------------------------------------------


def tt_apply_staged(x, cores) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    t = x.shape[0]
    z = x.reshape(t, 1, 1, -1)
    for g in cores:
        g = np.asarray(g, dtype=np.float64)
        a, mk, nk, b = g.shape
        i0 = z.shape[1]
        z = z.reshape(t, i0, a, nk, -1)
        z = np.einsum("tiajq,akjb->tikbq", z, g, optimize=True).reshape(t, i0 * mk, b, -1)
    return z.reshape(t, -1)


def tt_backward_staged(x, dy, cores):
    """(dx_adapter, [dG_k]) by the right-to-left stage walk (the GPU's qa_linear_backward order)."""
    x = np.asarray(x, dtype=np.float64)
    t = x.shape[0]
    cs = [np.asarray(g, dtype=np.float64) for g in cores]
    zs = [x.reshape(t, 1, 1, -1)]
    for g in cs[:-1]:
        a, mk, nk, b = g.shape
        z = zs[-1]
        i0 = z.shape[1]
        zs.append(np.einsum("tiajq,akjb->tikbq", z.reshape(t, i0, a, nk, -1), g, optimize=True)
                  .reshape(t, i0 * mk, b, -1))
    cur = np.asarray(dy, dtype=np.float64)
    grads = [None] * len(cs)
    for k in range(len(cs) - 1, -1, -1):
        g = cs[k]
        a, mk, nk, b = g.shape
        zin = zs[k]
        i0 = zin.shape[1]
        zin5 = zin.reshape(t, i0, a, nk, -1)
        dout5 = cur.reshape(t, i0, mk, b, -1)
        grads[k] = np.einsum("tiajq,tikbq->akjb", zin5, dout5, optimize=True)
        cur = np.einsum("tikbq,akjb->tiajq", dout5, g, optimize=True).reshape(t, -1)
    return cur.reshape(t, -1), grads


def qa_step_staged(x, dy, qw: OQuant, cores) -> dict:
    """One forward + backward of the quantised adapter linear on the CPU, staged (no W_t)."""
    x2 = np.asarray(x, dtype=np.float64).reshape(-1, qw.cols)
    qx = quantize_rows(x2, 8)
    y = qmatmul(qw, dequantize_rows(qx)) + tt_apply_staged(x2, cores)
    dxa, grads = tt_backward_staged(x2, dy, cores)
    dx = qmatmul_t(qw, dy) + dxa
    return {"y": y, "dx": dx, "dcores": grads}
