"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no LSTM, attention, softmax or
beam logic).  It only draws random numbers and writes/reads nothing but the
MNMT weight container and integer corpora, so that `oracle/` and the product
path can consume the same inputs without sharing any compute code.

Readings:
  * weights: numpy Generator(PCG64(seed)), ONE stream over the tensors in the
    canonical MNMT order (`tensor_specs`), uniform(-0.1, 0.1, shape) in fp64,
    cast to fp32 (BASELINE.json configs "weights U(-0.1,0.1)").
  * corpus: lengths uniform integers in [a, b] inclusive, drawn first; then ids.
    c1 ids are uniform in [4, V) (BASELINE.json configs[0]); c2..c5 ids are a
    truncated Zipf(s=1.1) over ranks r in [1, V-4], id = 3 + r, by inverse CDF.
  * ids 0..3 are reserved pad/unk/bos/eos (SPEC.md S170); pads are 0.
"""
from __future__ import annotations

import dataclasses
import os
import struct
from typing import Dict, List, Tuple

import numpy as np

PAD, UNK, BOS, EOS = 0, 1, 2, 3
MNMT_MAGIC = b"MNMT"
MNMT_VERSION = 1


@dataclasses.dataclass(frozen=True)
class ModelConfig:
    layers: int
    emb: int
    hidden: int          # decoder width == memory-bank width
    v_src: int
    v_tgt: int
    bidir: bool          # encoder bidirectional (per-direction width hidden/2)
    attn_general: bool   # 'general' (W_in present) vs 'dot'
    copy: bool = False   # copy / pointer generator: copy.w [1,H], copy.b [1]

    @property
    def h_dir(self) -> int:
        return self.hidden // 2 if self.bidir else self.hidden


@dataclasses.dataclass(frozen=True)
class DataConfig:
    batch: int
    len_lo: int
    len_hi: int
    zipf: bool           # Zipf(1.1) ids, else uniform in [4, V)
    fixed_lengths: Tuple[int, ...] = ()


@dataclasses.dataclass(frozen=True)
class DecodeConfig:
    beam: int
    max_len: int
    alpha: float
    precision: str       # "fp32" | "bf16"


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    model: ModelConfig
    data: DataConfig
    decode: DecodeConfig
    weight_seed: int = 0
    data_seed: int = 1


# BASELINE.json configs[0..4]; unstated values follow SURVEY.md AMB-28.
WORKLOADS: Dict[str, Workload] = {
    "c1": Workload("c1", ModelConfig(1, 32, 64, 100, 100, False, True),
                   DataConfig(2, 5, 8, False, fixed_lengths=(8, 5)),
                   DecodeConfig(3, 10, 0.0, "fp32")),
    "c2": Workload("c2", ModelConfig(2, 500, 500, 50000, 50000, False, True),
                   DataConfig(30, 10, 50, True),
                   DecodeConfig(5, 100, 0.0, "bf16")),
    "c3": Workload("c3", ModelConfig(2, 500, 500, 50000, 50000, True, False),
                   DataConfig(64, 20, 80, True),
                   DecodeConfig(5, 150, 0.0, "bf16")),
    "c4": Workload("c4", ModelConfig(4, 1000, 1000, 50000, 50000, False, True),
                   DataConfig(128, 10, 100, True),
                   DecodeConfig(5, 200, 0.6, "bf16")),
    "c5": Workload("c5", ModelConfig(2, 500, 512, 50000, 50000, True, True),
                   DataConfig(16, 300, 400, True),
                   DecodeConfig(10, 100, 0.0, "bf16")),
}


def tensor_specs(cfg: ModelConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    """Canonical MNMT tensor order and shapes (SURVEY.md §8(b) "Weight file")."""
    E, H, Hd, L = cfg.emb, cfg.hidden, cfg.h_dir, cfg.layers
    D = 2 if cfg.bidir else 1
    specs: List[Tuple[str, Tuple[int, ...]]] = [("enc.emb", (cfg.v_src, E))]
    for l in range(L):
        inp = E if l == 0 else D * Hd
        for d in (["fwd", "bwd"] if cfg.bidir else ["fwd"]):
            p = f"enc.l{l}.{d}."
            specs += [(p + "w_ih", (4 * Hd, inp)), (p + "w_hh", (4 * Hd, Hd)),
                      (p + "b_ih", (4 * Hd,)), (p + "b_hh", (4 * Hd,))]
    specs.append(("dec.emb", (cfg.v_tgt, E)))
    for l in range(L):
        inp = E + H if l == 0 else H
        p = f"dec.l{l}."
        specs += [(p + "w_ih", (4 * H, inp)), (p + "w_hh", (4 * H, H)),
                  (p + "b_ih", (4 * H,)), (p + "b_hh", (4 * H,))]
    if cfg.attn_general:
        specs.append(("attn.w_in", (H, H)))
    specs += [("attn.w_out", (H, 2 * H)), ("gen.w", (cfg.v_tgt, H)), ("gen.b", (cfg.v_tgt,))]
    if cfg.copy:
        specs += [("copy.w", (1, H)), ("copy.b", (1,))]
    return specs


def make_weights(cfg: ModelConfig, seed: int = 0) -> Dict[str, np.ndarray]:
    """U(-0.1, 0.1) fp32 weights from one PCG64 stream in canonical order (AMB-25)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out: Dict[str, np.ndarray] = {}
    for name, shape in tensor_specs(cfg):
        out[name] = rng.uniform(-0.1, 0.1, size=shape).astype(np.float32)
    return out


def write_mnmt(path: str, tensors: Dict[str, np.ndarray]) -> None:
    """SPEC.md S83 container: magic "MNMT", u32 version, then per tensor
    u32 name length + UTF-8 name, u32 rank, u64 dims, u32 dtype tag (f32=0),
    little-endian payload.  Read to EOF."""
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(MNMT_MAGIC)
        f.write(struct.pack("<I", MNMT_VERSION))
        for name, arr in tensors.items():
            a = np.ascontiguousarray(arr, dtype="<f4")
            nb = name.encode("utf-8")
            f.write(struct.pack("<I", len(nb)))
            f.write(nb)
            f.write(struct.pack("<I", a.ndim))
            f.write(struct.pack("<%dQ" % a.ndim, *a.shape))
            f.write(struct.pack("<I", 0))
            f.write(a.tobytes())
    os.replace(tmp, path)


def weights_file(workload: str, cache_dir: str, overrides: Dict[str, np.ndarray] | None = None,
                 tag: str = "") -> str:
    """Write (once) the MNMT file of a workload's model into cache_dir."""
    w = WORKLOADS[workload]
    os.makedirs(cache_dir, exist_ok=True)
    path = os.path.join(cache_dir, f"{workload}{('_' + tag) if tag else ''}_s{w.weight_seed}.mnmt")
    if not os.path.exists(path):
        t = make_weights(w.model, w.weight_seed)
        if overrides:
            t.update(overrides)
        write_mnmt(path, t)
    return path


def zipf_ids(rng: np.random.Generator, n: int, vocab: int, s: float = 1.1) -> np.ndarray:
    """Truncated Zipf over ranks 1..vocab-4, id = 3 + rank (AMB-26), inverse CDF."""
    ranks = np.arange(1, vocab - 4 + 1, dtype=np.float64)
    p = ranks ** (-s)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    u = rng.random(n)
    r = np.searchsorted(cdf, u, side="right") + 1
    r = np.minimum(r, vocab - 4)
    return (3 + r).astype(np.int32)


def make_corpus(workload: str, n_sentences: int | None = None, seed: int | None = None
                ) -> Tuple[np.ndarray, np.ndarray]:
    """Return (ids [N x S_max] int32 padded with 0, lens [N] int32).

    Lengths are drawn first (uniform integers in [a, b]), then ids (AMB-27)."""
    w = WORKLOADS[workload]
    d = w.data
    n = d.batch if n_sentences is None else n_sentences
    rng = np.random.Generator(np.random.PCG64(w.data_seed if seed is None else seed))
    if d.fixed_lengths and n == len(d.fixed_lengths):
        lens = np.array(d.fixed_lengths, dtype=np.int32)
    else:
        lens = rng.integers(d.len_lo, d.len_hi + 1, size=n).astype(np.int32)
    s_max = int(lens.max()) if n > 0 else 1
    ids = np.zeros((n, s_max), dtype=np.int32)
    for b in range(n):
        if d.zipf:
            ids[b, : lens[b]] = zipf_ids(rng, int(lens[b]), w.model.v_src)
        else:
            ids[b, : lens[b]] = rng.integers(4, w.model.v_src, size=int(lens[b]))
    return ids, lens


def random_model_tensors(cfg: ModelConfig, seed: int, scale: float = 0.1) -> Dict[str, np.ndarray]:
    """Toy models for tests: U(-scale, scale) in canonical order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return {n: rng.uniform(-scale, scale, size=s).astype(np.float32) for n, s in tensor_specs(cfg)}


def make_src_ext(ids: np.ndarray, lens: np.ndarray, v_tgt: int, seed: int = 5, p_shared: float = 0.7) -> np.ndarray:
    """Dynamic-dictionary input of the copy model (SPEC S293 "src_map: source-position ->
    extended-vocab-id"), as synthetic DATA: a seeded table decides which source ids have a
    target-vocabulary counterpart (the same id, when < v_tgt, with probability p_shared);
    every other distinct source id of a sentence gets the next extended id v_tgt, v_tgt+1, ...
    in order of first appearance.  Pads are 0."""
    rng = np.random.Generator(np.random.PCG64(seed))
    vmax = int(ids.max()) + 1 if ids.size else 1
    shared = rng.uniform(0, 1, vmax) < p_shared
    out = np.zeros_like(ids, dtype=np.int32)
    for b in range(len(lens)):
        extra: Dict[int, int] = {}
        for s in range(int(lens[b])):
            x = int(ids[b, s])
            if x < v_tgt and shared[x]:
                out[b, s] = x
            else:
                if x not in extra:
                    extra[x] = v_tgt + len(extra)
                out[b, s] = extra[x]
    return out
