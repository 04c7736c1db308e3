"""Device AdamW (qa_adamw_step) against the reference optimizer's own outputs
(tests/golden/adamw.npz from trainer.py:84-121 via oracle/gen_optim_golden.py): bit-identical float32
parameters and float64 masters after every step, and the non-finite-gradient error semantics."""

import os

import numpy as np
import pytest
import torch

from paper_2402_13533_b200 import optim
from paper_2402_13533_b200.linear import Param

pytestmark = pytest.mark.gpu


def _load():
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "adamw.npz"))
    names = sorted({k.split("__", 1)[1] for k in g.files if k.startswith("init__")})
    return g, names


def test_adamw_bit_identical_to_reference():
    g, names = _load()
    params = {k: Param(k, torch.from_numpy(g[f"init__{k}"]).cuda()) for k in names}
    state = optim.AdamWState(params)
    cfg = optim.AdamWConfig(lr=1e-3, weight_decay=0.05)
    for t in range(3):
        grads = {k: torch.from_numpy(g[f"g{t}__{k}"]).cuda() for k in names}
        optim.adamw_step(state, params, grads, cfg)
        for k in names:
            assert np.array_equal(params[k].data.cpu().numpy(), g[f"p{t}__{k}"]), (t, k)
            i = state.index[k]
            master = state.master[state.offsets[i]:state.offsets[i + 1]].cpu().numpy().reshape(g[f"w{t}__{k}"].shape)
            assert np.array_equal(master, g[f"w{t}__{k}"]), (t, k)


def test_adamw_nonfinite_gradient_names_tensor():
    g, names = _load()
    params = {k: Param(k, torch.from_numpy(g[f"init__{k}"]).cuda()) for k in names}
    state = optim.AdamWState(params)
    grads = {k: torch.from_numpy(g[f"g0__{k}"]).cuda() for k in names}
    grads[names[1]] = grads[names[1]].clone()
    grads[names[1]].view(-1)[3] = float("nan")
    before = {k: params[k].data.clone() for k in names}
    with pytest.raises(optim.TrainError, match=names[1]):
        optim.adamw_step(state, params, grads, optim.AdamWConfig())
    # sorted order: the tensor before the bad one was updated, the bad one and later ones were not
    assert not torch.equal(params[names[0]].data, before[names[0]])
    assert torch.equal(params[names[1]].data, before[names[1]])
    assert torch.equal(params[names[2]].data, before[names[2]])


def test_adamw_bound_flat_buffers_match_reference():
    """AdamWState.bind: parameters become views of the flat working copy and gradients are written into the
    flat gradient views (the decoder's path, no gather / copy-back) — still bit-identical to the reference."""
    g, names = _load()
    params = {k: Param(k, torch.from_numpy(g[f"init__{k}"]).cuda()) for k in names}
    state = optim.AdamWState(params)
    views = state.bind(params)
    for k in names:
        assert np.array_equal(params[k].data.cpu().numpy(), g[f"init__{k}"])
    cfg = optim.AdamWConfig(lr=1e-3, weight_decay=0.05)
    for t in range(3):
        for k in names:
            views[k].copy_(torch.from_numpy(g[f"g{t}__{k}"]))
        optim.adamw_step(state, params, views, cfg)
        for k in names:
            assert np.array_equal(params[k].data.cpu().numpy(), g[f"p{t}__{k}"]), (t, k)
