"""archive — the tensor_core ModelArchive: UTF-8 JSON manifest
behind an 8-byte little-endian header length (LEDGER G15), then a little-endian blob.
dtypes f32 | i8 | u4packed (two's-complement nibbles, low nibble = even index,
SPEC.md:32, 48, 74) | json-meta.  Weight names follow `blocks.<i>.<field>`.
Loading a quantized archive then repacks the u4 payload into the kernel layout once
(ssm_block.DeviceLinear -> sq_repack_w4).
"""
from __future__ import annotations

import json
import struct

import numpy as np

from .errors import ArchiveError, ShapeError

__all__ = ["pack_u4", "unpack_u4", "archive_write", "archive_read", "inspect", "write_float_model",
           "read_float_model", "write_quant_model", "read_quant_model"]


def pack_u4(vals) -> np.ndarray:
    v = np.asarray(vals)
    if v.shape[-1] % 2:
        raise ShapeError("u4packed needs an even last dimension")
    if v.size and (v.min() < -8 or v.max() > 7):
        raise ValueError("u4 values must lie in [-8, 7]")
    u = (v.astype(np.int64) & 0xF).astype(np.uint8)
    return (u[..., 0::2] | (u[..., 1::2] << 4)).astype(np.uint8)


def unpack_u4(packed) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.shape[:-1] + (p.shape[-1] * 2,), dtype=np.int8)
    out[..., 0::2] = ((p & 0xF).astype(np.int16) ^ 8) - 8
    out[..., 1::2] = ((p >> 4).astype(np.int16) ^ 8) - 8
    return out


def archive_write(tensors: dict, path: str) -> None:
    """SPEC.md:40-48.  Values: float32 / int8 arrays, ("u4packed", ints in [-8,7]) tuples,
    or JSON-serialisable metadata."""
    manifest, blobs, off = [], [], 0
    for name, v in tensors.items():
        if isinstance(v, tuple) and len(v) == 2 and v[0] == "u4packed":
            logical = np.asarray(v[1])
            payload = pack_u4(logical).tobytes()
            entry = {"name": name, "dtype": "u4packed", "shape": list(logical.shape)}
        elif isinstance(v, np.ndarray) and v.dtype == np.float32:
            if not np.isfinite(v).all():
                raise ArchiveError(f"{name} contains non-finite values")
            payload = v.astype("<f4").tobytes()
            entry = {"name": name, "dtype": "f32", "shape": list(v.shape)}
        elif isinstance(v, np.ndarray) and v.dtype == np.int8:
            payload = v.tobytes()
            entry = {"name": name, "dtype": "i8", "shape": list(v.shape)}
        else:
            payload = json.dumps(v, sort_keys=True).encode("utf-8")
            entry = {"name": name, "dtype": "json-meta", "shape": []}
        entry.update(byte_offset=off, byte_length=len(payload))
        manifest.append(entry)
        blobs.append(payload)
        off += len(payload)
    head = json.dumps(manifest, sort_keys=True).encode("utf-8")
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", len(head)))
        f.write(head)
        for b in blobs:
            f.write(b)


def archive_read(path: str) -> dict:
    """validates ordering, overlap, extent and finiteness."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise ArchiveError(f"cannot read archive: {e}") from e
    if len(raw) < 8:
        raise ArchiveError("archive shorter than header")
    (hl,) = struct.unpack("<Q", raw[:8])
    try:
        manifest = json.loads(raw[8:8 + hl].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise ArchiveError(f"corrupt manifest: {e}") from e
    blob = raw[8 + hl:]
    out, last_end, names = {}, 0, set()
    for e in sorted(manifest, key=lambda e: e["byte_offset"]):
        if e["name"] in names:
            raise ArchiveError(f"duplicate name {e['name']}")
        names.add(e["name"])
        if e["byte_offset"] < last_end:
            raise ArchiveError("overlapping ranges")
        end = e["byte_offset"] + e["byte_length"]
        if end > len(blob):
            raise ArchiveError("blob shorter than manifest extent")
        last_end = end
        b = blob[e["byte_offset"]:end]
        dt = e["dtype"]
        if dt == "json-meta":
            out[e["name"]] = json.loads(b.decode("utf-8"))
        elif dt == "u4packed":
            shp = tuple(e["shape"])
            out[e["name"]] = unpack_u4(np.frombuffer(b, np.uint8).reshape(shp[:-1] + (shp[-1] // 2,)))
        elif dt in ("f32", "i8"):
            a = np.frombuffer(b, "<f4" if dt == "f32" else np.int8).reshape(e["shape"]).copy()
            if dt == "f32":
                a = a.astype(np.float32)
                if not np.isfinite(a).all():
                    raise ArchiveError(f"{e['name']} contains non-finite values")
            out[e["name"]] = a
        else:
            raise ArchiveError(f"unknown dtype {dt}")
    return out


def inspect(path: str) -> dict:
    """Manifest summary (the `ssmquant inspect` subcommand)."""
    a = archive_read(path)
    return {k: (list(v.shape) + [str(v.dtype)] if isinstance(v, np.ndarray) else "json-meta") for k, v in a.items()}


# ------------------------------------------------------------------ model <-> archive
_BLOCK_F = ("in_proj", "conv_weight", "conv_bias", "a_log", "d_param", "dt_bias", "norm_weight", "out_proj",
            "x_proj", "dt_proj")


def write_float_model(fm, path: str) -> None:
    t = {"meta": {"kind": "float", "dims": vars(fm.dims), "n_blocks": len(fm.blocks)},
         "embedding": fm.embedding, "final_norm": fm.final_norm, "head": fm.head}
    for i, (ln, b) in enumerate(zip(fm.layer_norms, fm.blocks)):
        t[f"blocks.{i}.layer_norm"] = ln
        for f in _BLOCK_F:
            v = getattr(b, f)
            if v is not None:
                t[f"blocks.{i}.{f}"] = np.asarray(v, np.float32)
        if b.head_group is not None:
            t[f"blocks.{i}.head_group"] = np.asarray(b.head_group).tolist()
    archive_write(t, path)


def read_float_model(path: str):
    from .cli import FloatModel
    from .ssm_block import Dims, SsmBlockWeights
    a = archive_read(path)
    meta = a.get("meta", {})
    if meta.get("kind") != "float":
        raise ArchiveError("not a float-model archive")
    d = Dims(**meta["dims"])
    blocks, lns = [], []
    for i in range(meta["n_blocks"]):
        g = lambda f: a.get(f"blocks.{i}.{f}")   # noqa: E731
        hg = g("head_group")
        blocks.append(SsmBlockWeights(d, *[g(f) for f in _BLOCK_F[:8]], g("x_proj"), g("dt_proj"),
                                      np.asarray(hg, np.int32) if hg is not None else None))
        lns.append(g("layer_norm"))
    return FloatModel(d, a["embedding"], lns, blocks, a["final_norm"], a["head"])


def write_quant_model(qm, path: str) -> None:
    """Quantized model -> archive (SPEC.md:591 stage 11): u4packed payloads for 4-bit weights and
    embeddings, f32 scale tables, per-block scalars and the profile as json-meta."""
    emb_bits = int((getattr(qm, "extra", None) or {}).get("emb_bits", 8))
    t = {"meta": {"kind": "quantized", "dims": vars(qm.dims), "profiles": qm.profiles,
                  "s_head": float(qm.s_head), "emb_bits": emb_bits, "n_blocks": len(qm.blocks)},
         "emb_codes": ("u4packed", np.asarray(qm.emb_codes)) if emb_bits == 4 else np.asarray(qm.emb_codes, np.int8),
         "emb_scale": np.asarray(qm.emb_scale, np.float32), "final_norm": np.asarray(qm.final_norm, np.float32)}

    def put_ql(prefix, ql):
        t[f"{prefix}.meta"] = {"kind": ql.kind, "group": int(ql.group)}
        if ql.kind == "w8":
            t[f"{prefix}.codes"] = np.asarray(ql.codes, np.int8)
        else:
            t[f"{prefix}.codes"] = ("u4packed", np.asarray(ql.codes))
        for f in ("s_ch", "s_group"):
            if getattr(ql, f) is not None:
                t[f"{prefix}.{f}"] = np.asarray(getattr(ql, f), np.float32)

    put_ql("head", qm.head)
    for i, (ln, b) in enumerate(zip(qm.layer_norms, qm.blocks)):
        t[f"blocks.{i}.layer_norm"] = ln
        for f in ("in_proj", "out_proj", "x_proj", "dt_proj"):
            if getattr(b, f) is not None:
                put_ql(f"blocks.{i}.{f}", getattr(b, f))
        for f in ("conv_weight", "conv_bias", "a_log", "d_param", "dt_bias", "norm_weight", "in_out_scale",
                  "conv_in_scale", "conv_out_scale", "state_scale", "xproj_out_scale"):
            if getattr(b, f, None) is not None:
                t[f"blocks.{i}.{f}"] = np.asarray(getattr(b, f), np.float32)
        t[f"blocks.{i}.scalars"] = {"s_u": float(b.s_u), "s_y": float(b.s_y), "s_dt": float(b.s_dt),
                                    "hadamard": bool(b.hadamard), "profile": b.profile,
                                    "head_group": None if b.head_group is None else np.asarray(b.head_group).tolist()}
    archive_write(t, path)


def read_quant_model(path: str):
    """Archive written by ``write_quant_model`` -> cli.QuantModel (QuantizedMambaLM loads it and
    repacks the u4 payloads into the kernel layout once)."""
    from .cli import QuantModel
    from .ssm_block import Dims, QBlock, QLinear
    a = archive_read(path)
    meta = a.get("meta", {})
    if meta.get("kind") != "quantized":
        raise ArchiveError("not a quantized-model archive")
    d = Dims(**meta["dims"])

    def get_ql(prefix):
        m = a.get(f"{prefix}.meta")
        if m is None:
            return None
        codes = np.asarray(a[f"{prefix}.codes"], np.int8)
        return QLinear(m["kind"], codes, s_ch=a.get(f"{prefix}.s_ch"), s_group=a.get(f"{prefix}.s_group"),
                       group=int(m["group"]))

    n_blocks = int(meta.get("n_blocks", len(meta["profiles"])))
    blocks, lns = [], []
    for i in range(n_blocks):
        g = lambda f: a.get(f"blocks.{i}.{f}")   # noqa: E731
        sc = g("scalars")
        hg = sc.get("head_group")
        qb = QBlock(d, sc["profile"], get_ql(f"blocks.{i}.in_proj"), get_ql(f"blocks.{i}.out_proj"),
                    g("conv_weight"), g("conv_bias"), g("a_log"), g("d_param"), g("dt_bias"), g("norm_weight"),
                    None if hg is None else np.asarray(hg, np.int32), get_ql(f"blocks.{i}.x_proj"),
                    get_ql(f"blocks.{i}.dt_proj"), s_u=np.float32(sc["s_u"]), in_out_scale=g("in_out_scale"),
                    conv_in_scale=g("conv_in_scale"), conv_out_scale=g("conv_out_scale"),
                    state_scale=g("state_scale"), s_y=np.float32(sc["s_y"]), xproj_out_scale=g("xproj_out_scale"),
                    s_dt=np.float32(sc["s_dt"]), hadamard=bool(sc["hadamard"]))
        blocks.append(qb)
        lns.append(g("layer_norm"))
    return QuantModel(d, list(meta["profiles"]), np.asarray(a["emb_codes"], np.int8), a["emb_scale"], lns, blocks,
                      a["final_norm"], get_ql("head"), np.float32(meta["s_head"]),
                      extra={"emb_bits": int(meta.get("emb_bits", 8))})

