"""Oracle: SPEC `[MODULE] tensor_core` + shipped `tensor.py`.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``matmul`` restates `pkg/src/ssmquant/tensor.py:33-54` (ascending-k rank-1
  updates, float64 accumulate, float32 result).
* ``int_gemm`` is the exact integer GEMM the reference lacks:
  int8/int4 codes are multiplied in float64 BLAS, which is exact because every
  partial sum stays below 2**53.
* ``make_rng`` restates `tensor.py:57-69` with defect D1 fixed (Philox takes a
  2-word key): key=[seed, s0], counter=[s1, s2, 0, 0]  (LEDGER G1).
* ``pack_u4`` / ``unpack_u4``: SPEC.md:32,48,74 — signed two's-complement
  nibbles, low nibble = even index.
* ``archive_write`` / ``archive_read``: SPEC.md:28-57, 76 (JSON manifest with an
  8-byte LE header length, LEDGER G15).
"""
from __future__ import annotations

import json
import struct

import numpy as np


class ShapeError(ValueError):
    pass


def as_f32(x, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float32)
    if shape is not None:
        a = a.reshape(shape)
    return a


def require_finite(a, name="tensor"):
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{name} contains non-finite values")
    return a


def matmul(a, b) -> np.ndarray:
    """tensor.py:33-54 — c = a @ b, f64 accumulate in ascending k, f32 out."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim != 2 or b.ndim != 2:
        raise ShapeError(f"matmul needs 2-D operands, got {a.shape} and {b.shape}")
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ShapeError(f"inner dimensions disagree: {a.shape} x {b.shape}")
    a64 = a.astype(np.float64)
    b64 = b.astype(np.float64)
    acc = np.zeros((m, n), dtype=np.float64)
    for kk in range(k):
        acc += a64[:, kk:kk + 1] * b64[kk:kk + 1, :]
    return acc.astype(np.float32)


def matmul_fast(a, b) -> np.ndarray:
    """Float GEMM for large oracle runs: f64 BLAS, f32 out.

    Differs from ``matmul`` only in f64 summation order (≤1 ulp of f32 after
    rounding in practice); used where SPEC allows tolerance.
    """
    return (np.asarray(a, np.float64) @ np.asarray(b, np.float64)).astype(np.float32)


def int_gemm(a_codes, b_codes) -> np.ndarray:
    """Exact integer GEMM c[i,j] = sum_k a[i,k]*b[k,j] (int64 result).

    |a|,|b| <= 128 and K <= 2**30 keep every partial sum < 2**53, so float64
    BLAS is exact regardless of summation order.
    """
    a = np.asarray(a_codes)
    b = np.asarray(b_codes)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"int_gemm shapes {a.shape} x {b.shape}")
    c = a.astype(np.float64) @ b.astype(np.float64)
    return c.astype(np.int64)


def make_rng(seed: int, *stream: int) -> np.random.Generator:
    """tensor.py:57-69 with D1 fixed: Philox key=[seed, s0], counter=[s1, s2, 0, 0]."""
    if len(stream) > 3:
        raise ValueError("at most three substream keys are supported")
    s = [int(v) & 0xFFFFFFFFFFFFFFFF for v in stream] + [0, 0, 0]
    key = np.array([int(seed) & 0xFFFFFFFFFFFFFFFF, s[0]], dtype=np.uint64)
    counter = np.array([s[1], s[2], 0, 0], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key, counter=counter))


def pack_u4(vals) -> np.ndarray:
    """Pack signed ints in [-8, 7] two per byte along the last axis (low nibble = even)."""
    v = np.asarray(vals)
    if v.shape[-1] % 2:
        raise ShapeError("u4packed needs an even last dimension")
    if v.size and (v.min() < -8 or v.max() > 7):
        raise ValueError("u4 values must lie in [-8, 7]")
    u = (v.astype(np.int64) & 0xF).astype(np.uint8)
    return (u[..., 0::2] | (u[..., 1::2] << 4)).astype(np.uint8)


def unpack_u4(packed) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    lo = (p & 0xF).astype(np.int8)
    hi = (p >> 4).astype(np.int8)
    lo = np.where(lo > 7, lo - 16, lo).astype(np.int8)
    hi = np.where(hi > 7, hi - 16, hi).astype(np.int8)
    out = np.empty(p.shape[:-1] + (p.shape[-1] * 2,), dtype=np.int8)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    return out


# ---------------------------------------------------------------- archive
_DT = {"f32": np.float32, "i8": np.int8, "u4packed": np.uint8}


def archive_write(tensors: dict, path: str) -> None:
    """SPEC.md:40-48.  values: np.float32 / np.int8 arrays, ('u4packed', int-array)
    tuples (logical values in [-8,7]) or JSON-able metadata (dict/list/str)."""
    manifest, blobs, off = [], [], 0
    for name in tensors:
        v = tensors[name]
        if isinstance(v, tuple) and v[0] == "u4packed":
            logical = np.asarray(v[1])
            payload = pack_u4(logical).tobytes()
            entry = {"name": name, "dtype": "u4packed", "shape": list(logical.shape)}
        elif isinstance(v, np.ndarray) and v.dtype == np.float32:
            require_finite(v, name)
            payload = v.astype("<f4").tobytes()
            entry = {"name": name, "dtype": "f32", "shape": list(v.shape)}
        elif isinstance(v, np.ndarray) and v.dtype == np.int8:
            payload = v.tobytes()
            entry = {"name": name, "dtype": "i8", "shape": list(v.shape)}
        else:
            payload = json.dumps(v, sort_keys=True).encode("utf-8")
            entry = {"name": name, "dtype": "json-meta", "shape": []}
        entry["byte_offset"] = off
        entry["byte_length"] = len(payload)
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
    """SPEC.md:49-57."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 8:
        raise ValueError("archive shorter than header")
    (hl,) = struct.unpack("<Q", raw[:8])
    manifest = json.loads(raw[8:8 + hl].decode("utf-8"))
    blob = raw[8 + hl:]
    out, last_end, names = {}, 0, set()
    for e in sorted(manifest, key=lambda e: e["byte_offset"]):
        if e["name"] in names:
            raise ValueError(f"duplicate name {e['name']}")
        names.add(e["name"])
        if e["byte_offset"] < last_end:
            raise ValueError("overlapping ranges")
        end = e["byte_offset"] + e["byte_length"]
        if end > len(blob):
            raise ValueError("blob shorter than manifest extent")
        last_end = end
        b = blob[e["byte_offset"]:end]
        if e["dtype"] == "json-meta":
            out[e["name"]] = json.loads(b.decode("utf-8"))
        elif e["dtype"] == "u4packed":
            shp = tuple(e["shape"])
            out[e["name"]] = unpack_u4(np.frombuffer(b, np.uint8).reshape(shp[:-1] + (shp[-1] // 2,)))
        else:
            a = np.frombuffer(b, _DT[e["dtype"]]).reshape(e["shape"]).copy()
            if e["dtype"] == "f32":
                require_finite(a, e["name"])
            out[e["name"]] = a
    return out
