"""The reference's `LRLM` checkpoint container (pkg/src/lrlm/checkpoint.py) for the quantised-adapter path.

File layout (checkpoint.py:1-8): magic "LRLM" | version u32 LE | header length u64 LE | UTF-8 JSON header |
zero padding to 64 bytes | payload; every tensor starts 64-byte aligned in the payload, raw little-endian.
Quantised bases are "u8q" / "u4q" packed codes (4-bit: two per byte, low nibble = even column,
quant.py:37-52) with "<name>.scale" / "<name>.offset" float32 companions (checkpoint.py:64-70).

What this module adds for the device path:
  - `read_checkpoint` parses and validates a file exactly like the reference (`_read_header` :143-158,
    `_validate_table` :161-177) without building the numpy model;
  - `load_quantized` puts u8q / u4q codes straight into device buffers in the same layout (no
    re-quantisation), with the epilogue's Σcodes term from `qa_code_rowsum`;
  - `load_lora` / `load_tt` rebuild device adapters (`LoraLinear` under the reference's names
    "<slot>.base", "<slot>.down", "<slot>.up"; tensor-train cores under the new names "<slot>.core{k}"
    with their modes in the header's "tt_specs");
  - `save_checkpoint` writes the same deterministic layout (`save_checkpoint` :113-140), so entries read
    from a reference file and written back give a byte-identical file, and `collect_backends` serialises
    device backends (the reference's `_collect` :73-104 raises on backends it does not know).
"""

from __future__ import annotations

import io
import json
import os
import struct

import numpy as np
import torch

from . import _lib
from .linear import LoraLinear, QuantizedLinear, TTLinear, TTSpec, tt_merge
from .quant import QuantizedMatrix, _stream_ptr

__all__ = ["CheckpointError", "MAGIC", "VERSION", "ALIGN", "Checkpoint", "read_checkpoint", "quantized_from_arrays",
           "load_quantized",
           "load_lora", "load_tt", "save_checkpoint", "collect_backends"]

MAGIC = b"LRLM"
VERSION = 1
ALIGN = 64
# element type of each dtype tag (u8q / u4q payloads are packed code bytes)
_NP = {"f32": np.dtype("<f4"), "f16": np.dtype("<f2"), "u8q": np.dtype("<u1"), "u4q": np.dtype("<u1")}
# magic, version (u32 LE), header byte length (u64 LE)
_PREAMBLE = struct.Struct("<4sIQ")


def _align_up(n: int) -> int:
    return -(-n // ALIGN) * ALIGN


class CheckpointError(RuntimeError):
    """Same role as lrlm.checkpoint.CheckpointError."""


class Checkpoint:
    """A parsed file: `header` (dict), `table` (name -> dtype / shape / offset / length) and the raw bytes."""

    def __init__(self, data: bytes, header: dict, payload_start: int):
        self.data = data
        self.header = header
        self.table = header["tensors"]
        self.payload_start = payload_start

    def raw(self, name: str, expect=None) -> tuple[np.ndarray, dict]:
        ent = self.table.get(name)
        if ent is None:
            raise CheckpointError(f"checkpoint is missing tensor {name}")
        tags = (expect,) if isinstance(expect, str) else expect
        if tags is not None and ent["dtype"] not in tags:
            raise CheckpointError(f"{name}: stored as {ent['dtype']}, wanted one of {tags}")
        dt = _NP[ent["dtype"]]
        view = memoryview(self.data)[self.payload_start + ent["offset"]:][:ent["length"]]
        return np.frombuffer(view, dtype=dt), ent

    def array(self, name: str) -> np.ndarray:
        """A float tensor as float32 in its logical shape (f16 widened, like the reference's fetch)."""
        arr, ent = self.raw(name, ("f32", "f16"))
        return arr.reshape(ent["shape"]).astype(np.float32)

    def entries(self):
        """(name, dtype tag, logical shape, host array) in the file's (sorted) order — save_checkpoint's input."""
        return [(name, self.table[name]["dtype"], list(self.table[name]["shape"]), self.raw(name)[0])
                for name in sorted(self.table)]


def _parse_preamble(data: bytes) -> tuple[dict, int]:
    """Header dict and payload start of a file (the container layout of checkpoint.py:1-8)."""
    if len(data) < _PREAMBLE.size:
        raise CheckpointError("not a checkpoint: bad magic (file shorter than the preamble)")
    magic, version, hlen = _PREAMBLE.unpack_from(data)
    if magic != MAGIC:
        raise CheckpointError("not a checkpoint: bad magic")
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version} (this reader handles {VERSION})")
    end = _PREAMBLE.size + hlen
    if end > len(data):
        raise CheckpointError("truncated checkpoint: the JSON header runs past end of file")
    try:
        header = json.loads(bytes(data[_PREAMBLE.size:end]))
    except (UnicodeDecodeError, ValueError) as exc:
        raise CheckpointError(f"corrupt header: {exc}") from exc
    if not isinstance(header, dict) or not isinstance(header.get("tensors"), dict):
        raise CheckpointError("corrupt header: no tensor table")
    return header, _align_up(end)


def _check_table(table: dict, payload_len: int) -> None:
    """Every entry aligned, inside the payload, of a known dtype, with its quantisation companions; no two
    entries share bytes."""
    if not table:
        return
    names = list(table)
    starts = np.array([int(table[n]["offset"]) for n in names], dtype=np.int64)
    ends = starts + np.array([int(table[n]["length"]) for n in names], dtype=np.int64)
    for n, a, b in zip(names, starts, ends):
        tag = table[n]["dtype"]
        if tag not in _NP:
            raise CheckpointError(f"{n}: unknown dtype tag {tag!r}")
        if a % ALIGN != 0:
            raise CheckpointError(f"{n}: payload offset {a} is not a multiple of {ALIGN}")
        if a < 0 or b > payload_len:
            raise CheckpointError(f"{n}: tensor bytes [{a}, {b}) run past end of file (truncated?)")
        if tag in ("u8q", "u4q"):
            missing = [c for c in (n + ".scale", n + ".offset") if c not in table]
            if missing:
                raise CheckpointError(f"{n}: quantised tensor without its companion {missing[0]}")
    order = np.lexsort((ends, starts))
    clash = np.flatnonzero(starts[order][1:] < ends[order][:-1])
    if clash.size:
        first, second = names[order[clash[0]]], names[order[clash[0] + 1]]
        raise CheckpointError(f"tensors {first} and {second} share payload bytes")


def read_checkpoint(path) -> Checkpoint:
    with open(path, "rb") as f:
        data = f.read()
    header, payload_start = _parse_preamble(data)
    _check_table(header["tensors"], len(data) - payload_start)
    return Checkpoint(data, header, payload_start)


def _upload(arr: np.ndarray, dtype, device) -> torch.Tensor:
    host = torch.from_numpy(np.array(arr, copy=True)).pin_memory()
    return host.to(device=device, dtype=dtype, non_blocking=True)


def quantized_from_arrays(codes, scale, offset, rows: int, cols: int, bits: int, device="cuda") -> QuantizedMatrix:
    """A quantised base from the reference's host arrays (QuantizedMatrix fields, quant.py:55-70: u8 codes,
    4-bit packed two per byte, f32 scale / offset) into device buffers, codes byte for byte; the epilogue's
    Σcodes term from qa_code_rowsum."""
    if bits not in (4, 8):
        raise CheckpointError(f"bits must be 4 or 8, got {bits}")
    packed = (cols + 1) // 2 if bits == 4 else cols
    codes = np.asarray(codes, dtype=np.uint8)
    if codes.size != rows * packed:
        raise CheckpointError(f"{codes.size} code bytes for a {rows}x{cols} {bits}-bit grid")
    dev = torch.device(device)
    c = _upload(codes.reshape(rows, packed), torch.uint8, dev)
    sc = _upload(np.asarray(scale, dtype=np.float32).reshape(rows), torch.float32, dev)
    of = _upload(np.asarray(offset, dtype=np.float32).reshape(rows), torch.float32, dev)
    rowsum = torch.empty(rows, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().qa_code_rowsum(c.data_ptr(), rows, cols, bits, rowsum.data_ptr(), _stream_ptr(dev)),
               "qa_code_rowsum")
    return QuantizedMatrix(rows, cols, bits, c, sc, of, rowsum)


def load_quantized(ck: Checkpoint, name: str, device="cuda") -> QuantizedMatrix:
    """A u8q / u4q base straight into device buffers (checkpoint.py:186-197): codes byte for byte."""
    codes, ent = ck.raw(name, ("u8q", "u4q"))
    rows, cols = ent["shape"]
    bits = 4 if ent["dtype"] == "u4q" else 8
    packed = (cols + 1) // 2 if bits == 4 else cols
    if codes.size != rows * packed:
        raise CheckpointError(f"{name}: {codes.size} code bytes for a {rows}x{cols} {ent['dtype']} grid")
    return quantized_from_arrays(codes, ck.raw(name + ".scale", "f32")[0], ck.raw(name + ".offset", "f32")[0],
                                 rows, cols, bits, device)


def load_lora(ck: Checkpoint, slot: str, device="cuda") -> LoraLinear:
    """`<slot>.base` (quantised) + `<slot>.down` / `<slot>.up` -> device LoraLinear (checkpoint.py:208-216)."""
    base = QuantizedLinear(slot + ".base", load_quantized(ck, slot + ".base", device))
    down = torch.from_numpy(ck.array(slot + ".down")).to(device)
    up = torch.from_numpy(ck.array(slot + ".up")).to(device)
    return _honour_merged(ck, slot, LoraLinear(slot, base, down, up))


def _honour_merged(ck: Checkpoint, slot: str, adapter):
    """A slot the header marks merged is re-folded after loading, as the reference's load_checkpoint does
    (checkpoint.py:231-235)."""
    if ck.header.get("merged", {}).get(slot):
        tt_merge(adapter)
    return adapter


def load_tt(ck: Checkpoint, slot: str, device="cuda") -> TTLinear:
    """A tensor-train adapter saved by collect_backends: `<slot>.base` + `<slot>.core{k}`, modes in
    header["tt_specs"][slot]."""
    specs = ck.header.get("tt_specs", {})
    if slot not in specs:
        raise CheckpointError(f"{slot}: no tt_specs entry")
    sp = specs[slot]
    spec = TTSpec(tuple(sp["m"]), tuple(sp["n"]), tuple(sp["ranks"]))
    base = QuantizedLinear(slot + ".base", load_quantized(ck, slot + ".base", device))
    cores = [torch.from_numpy(ck.array(f"{slot}.core{k}")).to(device) for k in range(spec.d)]
    return _honour_merged(ck, slot, TTLinear(slot, base, spec, cores))


def _host(a) -> np.ndarray:
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


def save_checkpoint(path, entries, header: dict) -> None:
    """Deterministic writer of the reference layout (checkpoint.py:113-140): `entries` are (name, dtype tag,
    logical shape, array); `header` supplies every key but "tensors" (model_config, layer_specs, merged, …).
    Tensors go in name order, each at the next 64-byte boundary of the payload."""
    blobs = {name: (tag, list(shape), np.ascontiguousarray(_host(arr)).astype(_NP[tag], copy=False).tobytes())
             for name, tag, shape, arr in entries}
    table, cursor = {}, 0
    for name in sorted(blobs):
        tag, shape, raw = blobs[name]
        table[name] = {"dtype": tag, "shape": shape, "offset": cursor, "length": len(raw)}
        cursor = _align_up(cursor + len(raw))
    hdr = json.dumps({**header, "tensors": table}, sort_keys=True, separators=(",", ":")).encode("utf-8")
    head = _PREAMBLE.pack(MAGIC, VERSION, len(hdr)) + hdr
    buf = io.BytesIO()
    buf.write(head)
    buf.write(bytes(_align_up(len(head)) - len(head)))
    for name in sorted(blobs):
        raw = blobs[name][2]
        buf.write(raw)
        buf.write(bytes(_align_up(len(raw)) - len(raw)))
    out = buf.getvalue()
    # the last tensor's padding is part of the payload only up to the table's end (as in the reference)
    out = out[:_align_up(len(head)) + cursor]
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as f:
        f.write(out)
    os.replace(tmp, path)


def _quant_entries(name: str, q: QuantizedMatrix):
    h = q.to_numpy()
    return [(name, "u4q" if q.bits == 4 else "u8q", [q.rows, q.cols], h["codes"]),
            (name + ".scale", "f32", [q.rows], h["scale"]),
            (name + ".offset", "f32", [q.rows], h["offset"])]


def collect_backends(slots: dict):
    """(entries, header additions) for device backends keyed by slot path ("layers.0.wq", …): quantised
    bases as u8q / u4q, LoRA factors under the reference's names, TT cores as "<slot>.core{k}"."""
    entries, tt_specs, merged = [], {}, {}
    for path, b in slots.items():
        if isinstance(b, TTLinear) and b.merged:
            # the reference re-folds a merged slot on load with lora_merge, which refuses quantised bases
            # (checkpoint.py:231-235, lowrank.py:247-251): a merged adapter over codes has no LRLM encoding
            raise CheckpointError(f"{path}: save the adapter before merging it (merged adapters over quantised "
                                  "bases cannot be stored in an LRLM file)")
        if isinstance(b, LoraLinear):
            entries += _quant_entries(path + ".base", b.base.q)
            entries.append((b.down.name, "f32", list(b.down.data.shape), b.down.data))
            entries.append((b.up.name, "f32", list(b.up.data.shape), b.up.data))
            merged[path] = bool(b.merged)
        elif isinstance(b, TTLinear):
            entries += _quant_entries(path + ".base", b.base.q)
            for k, p in enumerate(b.cores):
                entries.append((f"{path}.core{k}", "f32", list(p.data.shape), p.data))
            tt_specs[path] = {"m": list(b.spec.m), "n": list(b.spec.n), "ranks": list(b.spec.ranks)}
            merged[path] = bool(b.merged)
        elif isinstance(b, QuantizedLinear):
            entries += _quant_entries(path, b.q)
        else:
            raise CheckpointError(f"{path}: cannot serialize backend {type(b).__name__}")
    extra = {"merged": merged}
    if tt_specs:
        extra["tt_specs"] = tt_specs
    return entries, extra
