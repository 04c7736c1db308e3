"""Data-parallel host logic on CPU: world_size 2 over gloo (127.0.0.1), mirroring the reference's
federated-round tests (pkg/tests/test_distsim.py:151-237): averaged gradients equal the
centralised gradient of the concatenated batch, only adapter tensors travel, divergent replicas
are rejected."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2402_13533_b200 import dp
from paper_2402_13533_b200.linear import Param, QuantizedLinear
from paper_2402_13533_b200.quant import QuantizedMatrix

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Replica:
    """The backend protocol (name, params()) over a CPU-resident quantised base."""

    def __init__(self, name, w, cores, bits=8):
        q = O.quantize_rows(w, bits)
        self.name = name
        self.q = QuantizedMatrix(q.rows, q.cols, bits, torch.from_numpy(q.codes), torch.from_numpy(q.scale),
                                 torch.from_numpy(q.offset), torch.from_numpy(q.rowsum().astype(np.int32)))
        self.base = QuantizedLinear(name + ".base", self.q)
        self.cores = [Param(f"{name}.core{k}", torch.from_numpy(c.astype(np.float32))) for k, c in enumerate(cores)]

    def params(self):
        return list(self.cores)


def _setup(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _worker_grads(rank, port, out):
    _setup(rank, port)
    try:
        shape = O.TTShape((1, 4, 8), (8, 2, 1), (1, 3, 3, 1))
        rng = np.random.default_rng(0)
        cores = [rng.standard_normal(shape.core_shape(k)) for k in range(shape.d)]
        x = rng.standard_normal((8, shape.K))
        dy = rng.standard_normal((8, shape.N))
        xs = dp.shard_tokens(torch.from_numpy(x), rank, WORLD).numpy()
        dys = dp.shard_tokens(torch.from_numpy(dy), rank, WORLD).numpy()
        _, g = O.tt_backward_staged(xs, dys, cores)
        grads = {f"w.core{k}": torch.from_numpy(gk.astype(np.float32)) for k, gk in enumerate(g)}
        dp.average_grads(grads)
        _, gfull = O.tt_backward_staged(x, dy, cores)
        for k, gk in enumerate(gfull):
            np.testing.assert_allclose(grads[f"w.core{k}"].numpy(), gk / WORLD, rtol=1e-5, atol=1e-6)
        # the payload is the adapter tensors only (test_distsim.py:188-205)
        flat, views = dp.flatten_grads(grads)
        assert flat.numel() == sum(int(np.prod(shape.core_shape(k))) for k in range(shape.d))
        out[rank] = 1
    finally:
        dist.destroy_process_group()


def _worker_divergence(rank, port, out):
    _setup(rank, port)
    try:
        w = O.seeded_random(16, 8, 3, std=0.02)
        cores = [np.full((1, 4, 8, 1), 0.5 + rank, np.float32)]  # rank-dependent adapter -> divergence
        same = [np.full((1, 4, 8, 1), 0.5, np.float32)]
        ok = _Replica("w", w, same)
        dp.check_replicas([ok])  # identical state passes
        bad = _Replica("w", w, cores)
        try:
            dp.check_replicas([bad])
            out[rank] = 0
        except dp.ReplicaDivergence:
            out[rank] = 1
    finally:
        dist.destroy_process_group()


def _worker_bench_layout(rank, port, out):
    """The exact exchange of bench.py and DecoderStack.train_step: every adapter-core gradient of the linear set
    lives in ONE flat buffer (dp.flat_views, linear order then core order), each rank fills its views from its
    own token shard — micro-batch by micro-batch, accumulating like the kernels' accumulate flag — and
    dp.average_flat_ (micro-batch mean, then the NCCL / gloo mean over replicas) leaves every view equal to the
    reference's average over all chunks (trainer.py:193-195, distsim.py:309-314)."""
    _setup(rank, port)
    try:
        rng = np.random.default_rng(1)
        linears = [("wq", O.TTShape((1, 2, 8), (4, 2, 1), (1, 3, 3, 1))),
                   ("wu", O.TTShape((1, 3, 8), (4, 2, 1), (1, 3, 3, 1))),
                   ("wd", O.TTShape((1, 2, 8), (6, 2, 1), (1, 3, 3, 1)))]
        cores = {nm: [rng.standard_normal(sh.core_shape(k)) for k in range(sh.d)] for nm, sh in linears}
        tokens, micro = 16, 2
        xs = {nm: rng.standard_normal((tokens, sh.K)) for nm, sh in linears}
        dys = {nm: rng.standard_normal((tokens, sh.N)) for nm, sh in linears}
        layout = [(f"{nm}.core{k}", sh.core_shape(k)) for nm, sh in linears for k in range(sh.d)]
        flat = torch.zeros(sum(int(np.prod(s)) for _, s in layout), dtype=torch.float32)
        views = dp.flat_views(flat, layout)
        for nm, sh in linears:
            x = dp.shard_tokens(torch.from_numpy(xs[nm]), rank, WORLD)
            dy = dp.shard_tokens(torch.from_numpy(dys[nm]), rank, WORLD)
            for mb in range(micro):  # micro-batches of this rank's shard
                part = slice(mb * x.shape[0] // micro, (mb + 1) * x.shape[0] // micro)
                _, g = O.tt_backward_staged(x[part].numpy(), dy[part].numpy(), cores[nm])
                for k, gk in enumerate(g):
                    views[f"{nm}.core{k}"] += torch.from_numpy(gk.astype(np.float32))
        dp.average_flat_(flat, micro)
        for nm, sh in linears:
            _, gfull = O.tt_backward_staged(xs[nm], dys[nm], cores[nm])
            for k, gk in enumerate(gfull):  # mean over WORLD * micro equal chunks
                np.testing.assert_allclose(views[f"{nm}.core{k}"].numpy(), gk / (WORLD * micro), rtol=1e-5,
                                           atol=1e-6)
        with pytest.raises(ValueError):
            dp.flat_views(flat, layout[:-1])
        out[rank] = 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("worker", [_worker_grads, _worker_divergence, _worker_bench_layout])
def test_two_rank_gloo(worker):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(worker, args=(port, out), nprocs=WORLD, join=True)
    assert dict(out) == {0: 1, 1: 1}


def test_shard_tokens_split_and_reassemble():
    b = torch.arange(24).reshape(8, 3)
    parts = [dp.shard_tokens(b, r, 4) for r in range(4)]
    assert torch.equal(torch.cat(parts), b)
    with pytest.raises(ValueError):
        dp.shard_tokens(b, 0, 3)


def test_single_process_average_is_identity():
    g = {"a": torch.ones(3), "b": torch.full((2, 2), 2.0)}
    dp.average_grads(g)
    assert torch.equal(g["a"], torch.ones(3)) and torch.equal(g["b"], torch.full((2, 2), 2.0))
