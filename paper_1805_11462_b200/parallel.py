"""Sentence-level data parallelism: one process per GPU, each rank
translates its own fixed-size slice of a corpus, hypotheses are gathered once with
`all_gather_into_tensor` (NCCL over NVLink on GPUs, gloo in the CPU tests).  No per-step
collectives exist - sentences are independent (SPEC S466, S483)."""
from __future__ import annotations

from typing import Dict, Tuple


def rank_slice(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [begin, end) block of sentences owned by `rank` (weak scaling: equal blocks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = n_total // world
    return rank * per, (rank + 1) * per


def gather_results(local: Dict[str, "torch.Tensor"], keys=("hyps", "lens", "scores")):
    """All-gather the per-rank result tensors (equal shapes on every rank) into
    [world * B, ...] tensors in rank order = corpus order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    out = {}
    for k in keys:
        t = local[k].contiguous()
        g = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(g, t)
        out[k] = g
    return out
