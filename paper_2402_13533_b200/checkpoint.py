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

import json
import os

import numpy as np
import torch

from . import _lib
from .linear import LoraLinear, QuantizedLinear, TTLinear, TTSpec
from .quant import QuantizedMatrix, _stream_ptr

__all__ = ["CheckpointError", "MAGIC", "VERSION", "ALIGN", "Checkpoint", "read_checkpoint", "quantized_from_arrays",
           "load_quantized",
           "load_lora", "load_tt", "save_checkpoint", "collect_backends"]

MAGIC = b"LRLM"
VERSION = 1
ALIGN = 64
_NP = {"f32": np.dtype("<f4"), "f16": np.dtype("<f2"), "u8q": np.dtype("<u1"), "u4q": np.dtype("<u1")}


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
        if name not in self.table:
            raise CheckpointError(f"checkpoint is missing tensor {name}")
        ent = self.table[name]
        if expect is not None and ent["dtype"] not in ((expect,) if isinstance(expect, str) else expect):
            raise CheckpointError(f"{name}: expected dtype {expect}, found {ent['dtype']}")
        a = self.payload_start + ent["offset"]
        return np.frombuffer(self.data, dtype=_NP[ent["dtype"]], count=ent["length"] // _NP[ent["dtype"]].itemsize,
                             offset=a), ent

    def array(self, name: str) -> np.ndarray:
        """A float tensor as float32 in its logical shape (f16 widened, like the reference's fetch)."""
        arr, ent = self.raw(name, ("f32", "f16"))
        return arr.reshape(ent["shape"]).astype(np.float32)

    def entries(self):
        """(name, dtype tag, logical shape, host array) in the file's (sorted) order — save_checkpoint's input."""
        out = []
        for name in sorted(self.table):
            arr, ent = self.raw(name)
            out.append((name, ent["dtype"], list(ent["shape"]), arr))
        return out


def read_checkpoint(path) -> Checkpoint:
    data = open(path, "rb").read()
    if len(data) < 16 or data[:4] != MAGIC:
        raise CheckpointError("not a checkpoint: bad magic")
    version = int.from_bytes(data[4:8], "little")
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}, expected {VERSION}")
    hlen = int.from_bytes(data[8:16], "little")
    if 16 + hlen > len(data):
        raise CheckpointError("truncated checkpoint: header runs past end of file")
    try:
        header = json.loads(data[16:16 + hlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise CheckpointError(f"corrupt header: {exc}") from exc
    payload_start = 16 + hlen + (-(16 + hlen)) % ALIGN
    table = header.get("tensors")
    if not isinstance(table, dict):
        raise CheckpointError("corrupt header: no tensor table")
    payload_len = len(data) - payload_start
    spans = []
    for name, ent in table.items():
        off, length = ent["offset"], ent["length"]
        if off % ALIGN:
            raise CheckpointError(f"{name}: offset {off} not {ALIGN}-byte aligned")
        if off < 0 or off + length > payload_len:
            raise CheckpointError(f"{name}: tensor bytes run past end of file (truncated?)")
        if ent["dtype"] not in _NP:
            raise CheckpointError(f"{name}: unknown dtype {ent['dtype']}")
        if ent["dtype"] in ("u8q", "u4q"):
            for companion in (name + ".scale", name + ".offset"):
                if companion not in table:
                    raise CheckpointError(f"{name}: missing companion tensor {companion}")
        spans.append((off, off + length, name))
    spans.sort()
    for (a0, a1, n1), (b0, _b1, n2) in zip(spans, spans[1:]):
        if b0 < a1:
            raise CheckpointError(f"overlapping tensors {n1} and {n2}")
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
    return LoraLinear(slot, base, down, up)


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
    return TTLinear(slot, base, spec, cores)


def _host(a) -> np.ndarray:
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


def save_checkpoint(path, entries, header: dict) -> None:
    """Deterministic writer of the reference layout (checkpoint.py:113-140): `entries` are (name, dtype tag,
    logical shape, array); `header` supplies every key but "tensors" (model_config, layer_specs, merged, …)."""
    entries = sorted(entries, key=lambda e: e[0])
    table, blobs, offset = {}, [], 0
    for name, tag, shape, array in entries:
        raw = np.ascontiguousarray(_host(array)).astype(_NP[tag], copy=False).tobytes()
        table[name] = {"dtype": tag, "shape": list(shape), "offset": offset, "length": len(raw)}
        blobs.append((offset, raw))
        offset += len(raw)
        offset += (-offset) % ALIGN
    full = dict(header)
    full["tensors"] = table
    hb = json.dumps(full, sort_keys=True, separators=(",", ":")).encode("utf-8")
    out = bytearray(MAGIC + VERSION.to_bytes(4, "little") + len(hb).to_bytes(8, "little") + hb)
    out += b"\x00" * ((-len(out)) % ALIGN)
    start = len(out)
    out += b"\x00" * offset
    for off, raw in blobs:
        out[start + off:start + off + len(raw)] = raw
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as f:
        f.write(bytes(out))
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
