"""FLOP v1 compressed checkpoints of FlashOptim state (mirror of
flashopt.checkpoint, byte-compatible in both directions).

Layout (reference: /root/reference/pkg/src/flashopt/checkpoint.py:1-23): a
24-byte little-endian header (magic "FLOP", u16 version 1, u8 kind, u8
optimizer tag, u64 step, u32 group size, u32 record count), the records
(u16 name length, UTF-8 name, u8 dtype tag, u8 rank, u64 dims, raw
little-endian payload) and a CRC32 of everything before it.  A flash state is
six records in a fixed order (checkpoint.py:111-123): weights.lp (bf16 bits),
weights.rho (i8 / i16), momentum.codes, momentum.scales (f16),
variance.codes, variance.scales.

The writer streams records straight from device memory in bounded pieces
with an incremental CRC, so an 8B-parameter state (~41 GB) never needs a
second host copy.  The reader applies the reference's validation and error
messages (CRC, truncation, magic, version, unknown tags, trailing bytes,
-128 / -32768 correction codes).

Beyond the reference (which writes one state per file): `save_optimizer` /
`load_optimizer` write one FLOP v1 file per parameter of a FlashAdamW /
FlashSGD / FlashLion plus a JSON manifest.
"""

from __future__ import annotations

import json
import os
import struct
import zlib
from typing import Iterable

import numpy as np
import torch

__all__ = ["CheckpointError", "save_checkpoint", "load_checkpoint", "inspect_checkpoint", "payload_bytes",
           "save_tensor_bundle", "load_tensor_bundle", "save_optimizer", "load_optimizer"]

MAGIC = b"FLOP"
VERSION = 1
KIND_REFERENCE, KIND_FLASH, KIND_BUNDLE = 0, 1, 2
KIND_NAMES = {KIND_REFERENCE: "reference", KIND_FLASH: "flash", KIND_BUNDLE: "bundle"}
OPTIMIZER_TAGS = {"sgd": 0, "adamw": 1, "lion": 2, None: 255}
OPTIMIZER_NAMES = {v: k for k, v in OPTIMIZER_TAGS.items()}
TAG_F32, TAG_BF16, TAG_F16, TAG_I8, TAG_U8, TAG_I16 = range(6)
TAG_DTYPES = {TAG_F32: np.dtype("<f4"), TAG_BF16: np.dtype("<u2"), TAG_F16: np.dtype("<f2"),
              TAG_I8: np.dtype("i1"), TAG_U8: np.dtype("u1"), TAG_I16: np.dtype("<i2")}
TAG_LABELS = {TAG_F32: "f32", TAG_BF16: "bf16", TAG_F16: "f16", TAG_I8: "i8", TAG_U8: "u8", TAG_I16: "i16"}
_PIECE = 1 << 26  # elements per device->host piece while writing


class CheckpointError(ValueError):
    """Malformed, truncated or corrupt checkpoint (checkpoint.py:69-70)."""


# ---------------------------------------------------------------------------
# writing
# ---------------------------------------------------------------------------
def _as_bytes_pieces(a) -> Iterable[bytes]:
    """Raw little-endian bytes of a flat torch / numpy array, in pieces."""
    if isinstance(a, torch.Tensor):
        t = a.detach().reshape(-1)
        if t.dtype == torch.bfloat16:
            t = t.view(torch.int16)
        elif t.dtype == torch.float16:
            t = t.view(torch.int16)
        for o in range(0, t.numel(), _PIECE):
            yield t[o:o + _PIECE].cpu().numpy().tobytes()
    else:
        arr = np.ascontiguousarray(a).reshape(-1)
        for o in range(0, arr.size, _PIECE):
            yield arr[o:o + _PIECE].tobytes()


class _CrcWriter:
    def __init__(self, fh):
        self.fh, self.crc, self.n = fh, 0, 0

    def write(self, b: bytes) -> None:
        self.fh.write(b)
        self.crc = zlib.crc32(b, self.crc)
        self.n += len(b)


def _numel(a) -> int:
    return int(a.numel()) if isinstance(a, torch.Tensor) else int(np.asarray(a).size)


def _record_header(name: str, tag: int, n: int) -> bytes:
    enc = name.encode("utf-8")
    return struct.pack("<H", len(enc)) + enc + struct.pack("<BBQ", tag, 1, n)  # rank-1 (n,), optim.py:154


def _flash_records(state) -> tuple[int, list]:
    """(group_size, [(name, tag, array)]) for a FlashState / HostFlashState."""
    from .host import HostFlashState

    if isinstance(state, HostFlashState):
        lp, rho, mq, ms, vq, vs = state.lp, state.rho, state.m_codes, state.m_scales, state.v_codes, state.v_scales
        gsz = state.group_size
        scheme = state.variance_scheme
    else:
        lp, rho = state.weights.lp_values, state.weights.corrections
        mq, ms = state.momentum.codes, state.momentum.scales
        vq = state.variance.codes if state.variance is not None else None
        vs = state.variance.scales if state.variance is not None else None
        gsz = state.momentum.spec.group_size
        scheme = state.variance_scheme
    if vq is not None and scheme != "companded":
        raise CheckpointError("unserializable state: linear-variance baseline states are not checkpointable")
    rho_i16 = (rho.dtype == torch.int16) if isinstance(rho, torch.Tensor) else (np.dtype(rho.dtype) == np.int16)
    m_u8 = (mq.dtype == torch.uint8) if isinstance(mq, torch.Tensor) else (np.dtype(mq.dtype) == np.uint8)
    recs = [("weights.lp", TAG_BF16, lp), ("weights.rho", TAG_I16 if rho_i16 else TAG_I8, rho),
            ("momentum.codes", TAG_U8 if m_u8 else TAG_I8, mq), ("momentum.scales", TAG_F16, ms)]
    if vq is not None:
        recs += [("variance.codes", TAG_U8, vq), ("variance.scales", TAG_F16, vs)]
    return gsz, recs


def _write(path, kind: int, optimizer, step: int, group_size: int, records: list) -> int:
    with open(path, "wb") as fh:
        w = _CrcWriter(fh)
        w.write(MAGIC + struct.pack("<HBBQII", VERSION, kind, OPTIMIZER_TAGS[optimizer], int(step), int(group_size),
                                    len(records)))
        for name, tag, arr in records:
            w.write(_record_header(name, tag, _numel(arr)))
            for piece in _as_bytes_pieces(arr):
                w.write(piece)
        fh.write(struct.pack("<I", w.crc))
        return w.n + 4


def save_checkpoint(state, path, optimizer: str | None = None) -> int:
    """Write one flash state (device FlashState or host HostFlashState);
    returns the byte count (checkpoint.py:134-144).  Without `optimizer`, the
    tag is inferred like the reference: adamw if a variance buffer exists,
    else sgd (so always pass optimizer="lion" for Lion states)."""
    gsz, recs = _flash_records(state)
    if optimizer is None:
        optimizer = "adamw" if len(recs) == 6 else "sgd"
    return _write(path, KIND_FLASH, optimizer, state.t, gsz, recs)


def save_tensor_bundle(tensors: dict, path, optimizer: str | None = None, step: int = 0) -> int:
    """Named float32 tensors (checkpoint.py:147-155)."""
    recs = []
    for name, a in tensors.items():
        a = a.detach().float().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float32)
        recs.append((name, TAG_F32, a))
    with open(path, "wb") as fh:
        w = _CrcWriter(fh)
        w.write(MAGIC + struct.pack("<HBBQII", VERSION, KIND_BUNDLE, OPTIMIZER_TAGS[optimizer], int(step), 0,
                                    len(recs)))
        for name, tag, a in recs:
            enc = name.encode("utf-8")
            w.write(struct.pack("<H", len(enc)) + enc + struct.pack("<BB", tag, a.ndim)
                    + b"".join(struct.pack("<Q", d) for d in a.shape))
            w.write(np.ascontiguousarray(a, dtype="<f4").tobytes())
        fh.write(struct.pack("<I", w.crc))
        return w.n + 4


# ---------------------------------------------------------------------------
# reading
# ---------------------------------------------------------------------------
def _parse(blob: bytes) -> dict:
    if len(blob) < 28:
        raise CheckpointError("truncated: shorter than the fixed header")
    if zlib.crc32(memoryview(blob)[:-4]) != struct.unpack_from("<I", blob, len(blob) - 4)[0]:
        raise CheckpointError("crc-mismatch: checkpoint is corrupt or truncated")
    end = len(blob) - 4
    if blob[:4] != MAGIC:
        raise CheckpointError("bad-magic: not a checkpoint file")
    version, kind, tag, step, gsz, count = struct.unpack_from("<HBBQII", blob, 4)
    if version != VERSION:
        raise CheckpointError(f"unsupported-version: {version}")
    if kind not in KIND_NAMES:
        raise CheckpointError(f"unknown payload kind: {kind}")
    if tag not in OPTIMIZER_NAMES:
        raise CheckpointError(f"unknown optimizer tag: {tag}")
    pos = 24
    records = []

    def need(k):
        if pos + k > end:
            raise CheckpointError("truncated: file ends inside a record")

    for _ in range(count):
        need(2)
        (nl,) = struct.unpack_from("<H", blob, pos)
        pos += 2
        need(nl)
        name = blob[pos:pos + nl].decode("utf-8")
        pos += nl
        need(2)
        dt, rank = struct.unpack_from("<BB", blob, pos)
        pos += 2
        if dt not in TAG_DTYPES:
            raise CheckpointError(f"unknown dtype tag: {dt}")
        need(8 * rank)
        dims = struct.unpack_from("<" + "Q" * rank, blob, pos) if rank else ()
        pos += 8 * rank
        n = int(np.prod(dims, dtype=np.int64)) if dims else 1
        nb = n * TAG_DTYPES[dt].itemsize
        need(nb)
        arr = np.frombuffer(blob, dtype=TAG_DTYPES[dt], count=n, offset=pos).reshape(dims)
        pos += nb
        records.append((name, dt, arr))
    if pos != end:
        raise CheckpointError("trailing bytes after the last tensor record")
    return {"kind": kind, "optimizer": OPTIMIZER_NAMES[tag], "step": step, "group_size": gsz, "records": records}


def _read(path) -> dict:
    with open(path, "rb") as fh:
        return _parse(fh.read())


def _validate_codes(name: str, tag: int, arr: np.ndarray) -> None:
    if tag == TAG_I8 and np.any(arr.view(np.uint8) == 0x80):
        raise CheckpointError(f"invalid-correction-code: {name} contains -128")
    if tag == TAG_I16 and np.any(arr.view(np.uint16) == 0x8000):
        raise CheckpointError(f"invalid-correction-code: {name} contains -32768")


def load_checkpoint(path, device=None):
    """Load a flash state, bit for bit (checkpoint.py:230-260).  With a
    `device` the result is a device FlashState, otherwise a HostFlashState
    (NumPy arrays, the reference's representation)."""
    from .host import HostFlashState

    parsed = _read(path)
    if parsed["kind"] == KIND_BUNDLE:
        raise CheckpointError("not a state checkpoint (tensor bundle); use load_tensor_bundle")
    recs = {name: (tag, arr) for name, tag, arr in parsed["records"]}
    if parsed["kind"] == KIND_REFERENCE:
        missing = {"theta", "m"} - recs.keys()
        if missing:
            raise CheckpointError(f"reference state missing tensors: {sorted(missing)}")
        return {"theta": recs["theta"][1], "m": recs["m"][1], "v": recs["v"][1] if "v" in recs else None,
                "t": int(parsed["step"])}
    missing = {"weights.lp", "weights.rho", "momentum.codes", "momentum.scales"} - recs.keys()
    if missing:
        raise CheckpointError(f"flash state missing tensors: {sorted(missing)}")
    for name, tag, arr in parsed["records"]:
        _validate_codes(name, tag, arr)
    gsz = parsed["group_size"] or 32
    get = lambda k: recs[k][1].reshape(-1).copy() if k in recs else None  # noqa: E731
    hs = HostFlashState(get("weights.lp").view(np.uint16), get("weights.rho"), get("momentum.codes"),
                        get("momentum.scales"), get("variance.codes"), get("variance.scales"),
                        int(parsed["step"]), gsz)
    if device is None:
        return hs
    from .formats import SplitTensor
    from .optim import FlashState
    from .quantize import GroupSpec, QuantizedState

    dev = torch.device(device)
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    spec = GroupSpec(gsz)
    w = SplitTensor(T(hs.lp.view(np.int16)).view(torch.bfloat16), T(hs.rho))
    m = QuantizedState(T(hs.m_codes), T(hs.m_scales), spec, "momentum")
    v = None
    if hs.v_codes is not None:
        v = QuantizedState(T(hs.v_codes), T(hs.v_scales), spec, "variance")
    return FlashState(w, m, v, hs.t)


def load_tensor_bundle(path) -> dict:
    parsed = _read(path)
    if parsed["kind"] != KIND_BUNDLE:
        raise CheckpointError("not a tensor bundle; use load_checkpoint")
    return {"optimizer": parsed["optimizer"], "step": int(parsed["step"]),
            "tensors": {name: arr.copy() for name, _, arr in parsed["records"]}}


def payload_bytes(path) -> dict:
    parsed = _read(path)
    rows = [{"name": n, "dtype_tag": t, "elements": int(a.size), "bytes": int(a.size * TAG_DTYPES[t].itemsize)}
            for n, t, a in parsed["records"]]
    return {"tensors": rows, "payload_bytes": sum(r["bytes"] for r in rows)}


def inspect_checkpoint(path) -> dict:
    parsed = _read(path)
    rows, weights = [], 0
    for n, t, a in parsed["records"]:
        rows.append({"name": n, "dtype": TAG_LABELS[t], "elements": int(a.size),
                     "bytes": int(a.size * TAG_DTYPES[t].itemsize)})
        if n in ("theta", "weights.lp"):
            weights = int(a.size)
    return {"kind": KIND_NAMES[parsed["kind"]], "optimizer": parsed["optimizer"], "step": int(parsed["step"]),
            "group_size": int(parsed["group_size"]), "tensor_count": len(rows), "tensors": rows,
            "payload_bytes": sum(r["bytes"] for r in rows), "params": weights}


# ---------------------------------------------------------------------------
# whole optimizers: one FLOP v1 file per parameter + manifest
# ---------------------------------------------------------------------------
def save_optimizer(optimizer, directory, names: list[str] | None = None) -> dict:
    """Write every parameter's state of a FlashAdamW / FlashSGD / FlashLion as
    FLOP v1 (the bf16 weights are the state's weights.lp record)."""
    os.makedirs(directory, exist_ok=True)
    params = [p for g in optimizer.param_groups for p in g["params"]]
    names = names or [f"param{i:05d}" for i in range(len(params))]
    manifest = {"format": "FLOP v1 per parameter", "optimizer": optimizer.OPT, "params": []}
    total = 0
    for i, (p, name) in enumerate(zip(params, names)):
        fname = f"{i:05d}.flop"
        total += save_checkpoint(optimizer.flash_state(p), os.path.join(directory, fname), optimizer.OPT)
        manifest["params"].append({"index": i, "name": name, "file": fname, "shape": list(p.shape)})
    manifest["bytes"] = total
    with open(os.path.join(directory, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    return manifest


def load_optimizer(optimizer, directory) -> None:
    """Restore parameters (bf16 weights.lp) and optimizer state written by save_optimizer."""
    with open(os.path.join(directory, "manifest.json")) as f:
        manifest = json.load(f)
    if manifest["optimizer"] != optimizer.OPT:
        raise CheckpointError(f"checkpoint is for {manifest['optimizer']}, optimizer is {optimizer.OPT}")
    params = [p for g in optimizer.param_groups for p in g["params"]]
    if len(params) != len(manifest["params"]):
        raise CheckpointError("parameter count differs from the checkpoint")
    if hasattr(optimizer, "_plans"):
        optimizer._plans = {}  # cached launch tables point at the replaced state tensors
    with torch.no_grad():
        for p, ent in zip(params, manifest["params"]):
            if list(p.shape) != ent["shape"]:
                raise CheckpointError(f"shape mismatch for {ent['name']}")
            fs = load_checkpoint(os.path.join(directory, ent["file"]), device=p.device)
            rec = {"weights.rho": fs.weights.corrections, "momentum.scales": fs.momentum.scales}
            if fs.variance is not None:
                rec["variance.scales"] = fs.variance.scales
            if hasattr(optimizer, "_check_layout"):
                try:
                    optimizer._check_layout(p, rec)
                except ValueError as e:
                    raise CheckpointError(f"{ent['name']}: {e}") from None
            if p.dtype != torch.bfloat16:
                p.data = torch.empty(p.shape, dtype=torch.bfloat16, device=p.device)
            p.data.view(-1).copy_(fs.weights.lp_values)
            st = optimizer.state[p]
            st["weights.rho"] = fs.weights.corrections.view(p.shape).clone()
            st["momentum.codes"] = fs.momentum.codes.view(p.shape).clone()
            st["momentum.scales"] = fs.momentum.scales.clone()
            if fs.variance is not None:
                st["variance.codes"] = fs.variance.codes.view(p.shape).clone()
                st["variance.scales"] = fs.variance.scales.clone()
            st["step"] = fs.t
    if hasattr(optimizer, "_reset_capturable"):
        optimizer._reset_capturable()
