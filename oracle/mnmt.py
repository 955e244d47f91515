"""MNMT weight container reader and bf16 rounding (oracle side).

SPEC.md S83: magic "MNMT", u32 format version, then per tensor: u32 name length
+ UTF-8 name, u32 rank, u64 dims[rank], u32 dtype tag (f32 = 0), little-endian
payload; read to EOF.

O1 / AMB-23: in bf16 mode every tensor is rounded to bf16 with
round-to-nearest-even, exactly (the result is an fp32 value held in fp64), and
the oracle then evaluates THOSE weights in fp64.
"""
from __future__ import annotations

import struct
from typing import Dict

import numpy as np


def read_mnmt(path: str) -> Dict[str, np.ndarray]:
    """Parse an MNMT file into name -> float32 array (S83)."""
    out: Dict[str, np.ndarray] = {}
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"MNMT":
        raise ValueError("bad magic")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != 1:
        raise ValueError("unsupported MNMT version %d" % version)
    off = 8
    while off < len(data):
        (nlen,) = struct.unpack_from("<I", data, off); off += 4
        name = data[off:off + nlen].decode("utf-8"); off += nlen
        (rank,) = struct.unpack_from("<I", data, off); off += 4
        dims = struct.unpack_from("<%dQ" % rank, data, off); off += 8 * rank
        (tag,) = struct.unpack_from("<I", data, off); off += 4
        if tag != 0:
            raise ValueError("unsupported dtype tag %d" % tag)
        n = int(np.prod(dims)) if rank else 1
        arr = np.frombuffer(data, dtype="<f4", count=n, offset=off).reshape(dims)
        off += 4 * n
        out[name] = arr.copy()
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returns float32.

    bf16 keeps the top 16 bits of the IEEE-754 binary32 pattern.  RNE: add
    0x7FFF plus the lowest kept bit, then truncate.  (Finite inputs only.)"""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    keep_lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + keep_lsb) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32)


def load_model_tensors(path: str, precision: str) -> Dict[str, np.ndarray]:
    """O1: read the file; in bf16 mode round every tensor to bf16; return fp64."""
    raw = read_mnmt(path)
    if precision not in ("fp32", "bf16"):
        raise ValueError(precision)
    out = {}
    for k, v in raw.items():
        if precision == "bf16":
            v = bf16_round(v)
        out[k] = v.astype(np.float64)
    return out
