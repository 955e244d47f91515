"""Sentence-level data parallelism: one process per GPU, each rank translates
its own sentences, and the results are gathered once with `all_gather_into_tensor` (NCCL over
NVLink on GPUs, gloo in the CPU tests).  No per-step collectives exist - sentences are
independent (SPEC S466, S483; PAPER.md P219-224 names data parallelism across GPUs).

Two partitionings:
  * corpus mode: batches are formed deterministically in corpus order (fixed size, the last
    one ragged) and dealt round-robin to the ranks (`deal_batches`) - every batch has the
    same composition whatever the GPU count;
  * one batch sharded by sentence (`rank_slice`, strong scaling of c3 / c5): contiguous
    blocks, the remainder going to the first ranks.
The gather carries every output (hypotheses, lengths, normalised and raw scores, token
log-probabilities) plus the ORIGINAL sentence index of each row; ranks pad to the largest
local count and `gather_results` restores corpus order.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

RESULT_KEYS = ("hyps", "lens", "scores", "raw", "token_logp")


def rank_slice(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [begin, end) block of sentences owned by `rank`; the n_total % world
    leftover sentences go one each to the first ranks (no sentence is dropped)."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError("bad world/rank/n_total")
    per, extra = divmod(n_total, world)
    b0 = rank * per + min(rank, extra)
    return b0, b0 + per + (1 if rank < extra else 0)


def make_batches(n_sentences: int, batch: int) -> List[Tuple[int, int]]:
    """Corpus-order batches [begin, end) of `batch` sentences (the last one ragged)."""
    if batch < 1 or n_sentences < 0:
        raise ValueError("bad batch/n_sentences")
    return [(s, min(s + batch, n_sentences)) for s in range(0, n_sentences, batch)]


def deal_batches(n_batches: int, world: int, rank: int) -> List[int]:
    """Round-robin deal: batch i goes to rank i % world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_batches, world))


def gather_results(local: Dict[str, "torch.Tensor"], index: "torch.Tensor", keys: Sequence[str] = RESULT_KEYS,
                   n_total: int | None = None):
    """All-gather every rank's results (rows = local sentences, any count per rank) and
    their original sentence indices; returns {key: tensor [n_total, ...]} in corpus order
    on every rank.  One size exchange plus one all_gather_into_tensor per key."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = index.device
    n_local = torch.tensor([index.numel()], dtype=torch.int64, device=dev)
    sizes = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, n_local)
    sizes_l = [int(v) for v in sizes.cpu()]
    n_max = max(sizes_l)
    total = sum(sizes_l) if n_total is None else n_total

    def padded(t):
        t = t.contiguous()
        if t.shape[0] == n_max:
            return t
        p = torch.zeros((n_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        p[:t.shape[0]] = t
        return p

    gi = torch.empty(world * n_max, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(gi, padded(index.to(torch.int64)))
    valid = torch.cat([torch.arange(r * n_max, r * n_max + sizes_l[r], device=dev) for r in range(world)])
    order = gi[valid]
    out = {}
    for k in keys:
        t = padded(local[k])
        g = torch.empty((world * n_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(g, t)
        res = torch.zeros((total,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        res[order] = g[valid]
        out[k] = res
    return out


def translate_batches(model, ids, lens, batches: Sequence[Tuple[int, int]], mine: Sequence[int], beam: int,
                      max_len: int, length_penalty: float = 0.0):
    """Host-API translation of this rank's batches (numpy in, numpy out) with the original
    sentence index of every row; each batch is trimmed to its own longest source."""
    import numpy as np
    outs, idx = [], []
    for i in mine:
        b0, b1 = batches[i]
        L = lens[b0:b1]
        S = int(L.max())
        outs.append(model.translate(np.ascontiguousarray(ids[b0:b1, :S]), L, beam, max_len, length_penalty))
        idx.append(np.arange(b0, b1))
    if not outs:
        z = {"hyps": np.zeros((0, max_len), np.int32), "lens": np.zeros(0, np.int32),
             "scores": np.zeros(0, np.float32), "raw": np.zeros(0, np.float32),
             "token_logp": np.zeros((0, max_len), np.float32)}
        return z, np.zeros(0, np.int64)
    return {k: np.concatenate([o[k] for o in outs]) for k in RESULT_KEYS}, np.concatenate(idx)


def open_vocab_parallel(model, max_rows: int, group=None):
    """Vocabulary-parallel generator: every rank allocates its exchange
    buffer, the IPC handles are all-gathered (one object collective at set-up, not per step) and
    every rank maps the others' buffers.  Afterwards each rank's translate calls stream 1/world of
    W_gen and exchange the generator partials through peer memory inside the decode graph; every
    rank returns the same translation."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = model.vp_handle(max_rows)
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    if any(h is None or len(h) != 64 for h in handles):
        raise RuntimeError("bad exchange handle")
    model.vp_open(world, rank, b"".join(handles))
    return world, rank
