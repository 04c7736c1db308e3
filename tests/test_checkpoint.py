"""The LRLM checkpoint container against files written by the reference's own save_checkpoint
(tests/golden/ckpt_small.lrlm, made by oracle/gen_checkpoint_golden.py): parsing, validation errors,
byte-identical re-serialisation (CPU), and device loading of u8q / u4q bases and adapters (GPU)."""

import os

import numpy as np
import pytest
import torch

from paper_2402_13533_b200 import checkpoint as ckpt

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FILE = os.path.join(GOLD, "ckpt_small.lrlm")


def _golden():
    return np.load(os.path.join(GOLD, "ckpt_small.npz"))


def test_reader_matches_reference_arrays():
    ck = ckpt.read_checkpoint(FILE)
    g = _golden()
    assert ck.header["model_config"]["dim"] == 64
    for name in ("wq", "wk", "wv", "wo", "wu", "wg", "wd"):
        slot = f"layers.0.{name}"
        qname = slot + ".base" if name in ("wq", "wv", "wu") else slot
        codes, ent = ck.raw(qname)
        bits = int(g[f"{name}.bits"])
        assert ent["dtype"] == ("u4q" if bits == 4 else "u8q")
        assert np.array_equal(codes.reshape(g[f"{name}.codes"].shape), g[f"{name}.codes"])
        assert np.array_equal(ck.raw(qname + ".scale")[0], g[f"{name}.scale"])
        assert np.array_equal(ck.raw(qname + ".offset")[0], g[f"{name}.offset"])
    for name in ("wq", "wv", "wu"):
        assert np.array_equal(ck.array(f"layers.0.{name}.down"), g[f"{name}.down"])
        assert np.array_equal(ck.array(f"layers.0.{name}.up"), g[f"{name}.up"])


def test_writer_is_byte_identical(tmp_path):
    ck = ckpt.read_checkpoint(FILE)
    header = {k: v for k, v in ck.header.items() if k != "tensors"}
    out = tmp_path / "copy.lrlm"
    ckpt.save_checkpoint(out, ck.entries(), header)
    assert open(out, "rb").read() == open(FILE, "rb").read()


def test_validation_errors(tmp_path):
    data = open(FILE, "rb").read()
    bad = tmp_path / "bad.lrlm"
    bad.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(ckpt.CheckpointError, match="magic"):
        ckpt.read_checkpoint(bad)
    bad.write_bytes(data[:4] + (2).to_bytes(4, "little") + data[8:])
    with pytest.raises(ckpt.CheckpointError, match="version"):
        ckpt.read_checkpoint(bad)
    bad.write_bytes(data[: len(data) - 100])
    with pytest.raises(ckpt.CheckpointError, match="truncated|past end"):
        ckpt.read_checkpoint(bad)
    ck = ckpt.read_checkpoint(FILE)
    with pytest.raises(ckpt.CheckpointError, match="missing tensor"):
        ck.raw("layers.0.nope")


@pytest.mark.gpu
def test_device_loading_and_roundtrip(tmp_path):
    import oracle as O
    import paper_2402_13533_b200 as qa
    from paper_2402_13533_b200 import linear as L

    ck = ckpt.read_checkpoint(FILE)
    g = _golden()
    for name, slot in (("wk", "layers.0.wk"), ("wd", "layers.0.wd")):
        q = ckpt.load_quantized(ck, slot)
        assert np.array_equal(q.codes.cpu().numpy(), g[f"{name}.codes"])
        unpacked = q.unpacked_codes().cpu().numpy().astype(np.int64)
        assert np.array_equal(q.rowsum.cpu().numpy(), unpacked.sum(axis=1))
        # the loaded base computes exactly what the reference's stored codes mean (qmatmul, quant.py:123-132)
        x = O.seeded_random(9, q.cols, 4)
        oq = O.OQuant(q.rows, q.cols, q.bits, g[f"{name}.codes"], g[f"{name}.scale"], g[f"{name}.offset"])
        want = O.qmatmul(oq, O.dequantize_rows(O.quantize_rows(x, 8)))
        assert O.rel_err(qa.qmatmul(q, torch.from_numpy(x).cuda(), act_quant=True).cpu().numpy(), want) <= 1e-5
        assert O.rel_err(qa.qmatmul(q, torch.from_numpy(x).cuda()).cpu().numpy(), O.qmatmul(oq, x)) <= 1e-5
    lora = ckpt.load_lora(ck, "layers.0.wq")
    assert torch.equal(lora.down.data.cpu(), torch.from_numpy(g["wq.down"]))
    # device backends -> file -> device backends (LoRA under the reference's names, TT cores under new ones)
    base = L.QuantizedLinear("t.base", ckpt.load_quantized(ck, "layers.0.wu.base"))
    spec = L.TTSpec((1, 96), (16, 4), (1, 4, 1))
    tt = L.attach_tt_adapter("layers.0.wu", base, r=4, spec=spec, seed=2)
    entries, extra = ckpt.collect_backends({"layers.0.wq": lora, "layers.0.wu": tt, "layers.0.wk": L.QuantizedLinear(
        "layers.0.wk", ckpt.load_quantized(ck, "layers.0.wk"))})
    path = tmp_path / "dev.lrlm"
    ckpt.save_checkpoint(path, entries, extra)
    ck2 = ckpt.read_checkpoint(path)
    tt2 = ckpt.load_tt(ck2, "layers.0.wu")
    for a, b in zip(tt.cores, tt2.cores):
        assert torch.equal(a.data, b.data)
    assert torch.equal(tt2.base.q.codes, tt.base.q.codes)
    x = torch.from_numpy(O.seeded_random(5, 64, 8)).cuda().to(torch.bfloat16)
    assert torch.equal(tt.forward(x), tt2.forward(x))
    l2 = ckpt.load_lora(ck2, "layers.0.wq")
    assert torch.equal(l2.up.data, lora.up.data) and torch.equal(l2.base.q.codes, lora.base.q.codes)
