"""Data parallelism for the quantised tensor-adapter linear: one process per GPU, token batch
sharded by sequence, adapter gradients averaged with one all-reduce.

This is the real-collective version of the reference's in-process federated round
(lrlm/distsim.py:279-331): replicas must start identical (state_signature check,
distsim.py:293-296 / transformer.py:735-747), every rank runs forward + backward on its own
shard, and the gradients of the trainable tensors are summed in a fixed order and divided by
the replica count (distsim.py:309-314).  Only adapter tensors travel (the `lora` mode payload
contract, pkg/tests/test_distsim.py:188-205); the frozen quantised base never moves.

On NCCL the flat fp32 buffer is reduced with one ncclAllReduce over NVLink/NVSwitch (NVLS
when available); on gloo (CPU tests) the same code path runs over TCP.
"""

from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist

__all__ = [
    "ReplicaDivergence",
    "shard_tokens",
    "flatten_grads",
    "allreduce_mean_",
    "average_flat_",
    "flat_views",
    "average_grads",
    "state_signature",
    "check_replicas",
]


class ReplicaDivergence(ValueError):
    """Same role as the reference's ModelError('replica divergence ...') (distsim.py:293-296)."""


def _world(group=None):
    return dist.get_world_size(group) if dist.is_initialized() else 1


def _rank(group=None):
    return dist.get_rank(group) if dist.is_initialized() else 0


def shard_tokens(batch: torch.Tensor, rank: int | None = None, world: int | None = None) -> torch.Tensor:
    """This rank's equal share of a [sequences, ...] batch (sequences split contiguously)."""
    rank = _rank() if rank is None else rank
    world = _world() if world is None else world
    n = batch.shape[0]
    if n % world:
        raise ValueError(f"{n} sequences do not split evenly over {world} ranks")
    per = n // world
    return batch[rank * per:(rank + 1) * per]


def flatten_grads(grads: dict, names=None):
    """One contiguous fp32 buffer holding `grads` in sorted-name order, plus the views into it."""
    names = sorted(grads) if names is None else list(names)
    ref = grads[names[0]]
    total = sum(grads[n].numel() for n in names)
    flat = torch.empty(total, dtype=torch.float32, device=ref.device)
    views, off = {}, 0
    for n in names:
        g = grads[n]
        v = flat[off:off + g.numel()]
        v.copy_(g.reshape(-1).float())
        views[n] = v.view(g.shape)
        off += g.numel()
    return flat, views


def allreduce_mean_(flat: torch.Tensor, group=None) -> torch.Tensor:
    """In-place mean over ranks: one SUM all-reduce then x 1/G (distsim.py:309-314)."""
    world = _world(group)
    if world > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        flat.mul_(1.0 / world)
    return flat


def flat_views(flat: torch.Tensor, named_shapes) -> dict:
    """Views of one contiguous gradient buffer, laid out in the given (name, shape) order — the layout the
    bench and the training step reduce with a single collective."""
    views, off = {}, 0
    for name, shape in named_shapes:
        n = 1
        for d in shape:
            n *= int(d)
        views[name] = flat[off:off + n].view(*shape)
        off += n
    if off != flat.numel():
        raise ValueError(f"layout covers {off} of {flat.numel()} elements")
    return views


def average_flat_(flat: torch.Tensor, micro_batches: int = 1, group=None) -> torch.Tensor:
    """The gradient exchange of one training step on a flat buffer, in place: the micro-batch average of
    trainer.train_step (trainer.py:193-195), then the mean over the data-parallel replicas
    (distsim.federated_round, distsim.py:309-314)."""
    if micro_batches > 1:
        flat.div_(micro_batches)
    return allreduce_mean_(flat, group)


def average_grads(grads: dict, group=None) -> dict:
    """Average a grads dict (name -> tensor) over the data-parallel group, in place."""
    if not grads:
        return grads
    flat, views = flatten_grads(grads)
    allreduce_mean_(flat, group)
    for n, v in views.items():
        grads[n].copy_(v.view_as(grads[n]))
    return grads


def state_signature(backends) -> bytes:
    """sha256 over every backend's quantised codes / scales / offsets and adapter tensors
    (the reference's DecoderModel.state_signature, transformer.py:735-747)."""
    h = hashlib.sha256()
    for b in backends:
        h.update(b.name.encode())
        q = getattr(b, "q", None) or getattr(getattr(b, "base", None), "q", None)
        if q is not None:
            for t in (q.codes, q.scale, q.offset):
                h.update(t.detach().cpu().numpy().tobytes())
        for p in b.params():
            h.update(p.name.encode())
            h.update(p.data.detach().cpu().float().numpy().tobytes())
    return h.digest()


def check_replicas(backends, group=None) -> bytes:
    """Raise ReplicaDivergence unless every rank holds byte-identical state."""
    sig = state_signature(backends)
    world = _world(group)
    if world == 1:
        return sig
    mine = torch.tensor(list(sig), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        mine = mine.cuda()
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    for i, g in enumerate(gathered):
        if not torch.equal(g.cpu(), mine.cpu()):
            raise ReplicaDivergence(f"replica divergence detected at round start (rank {i})")
    return sig
