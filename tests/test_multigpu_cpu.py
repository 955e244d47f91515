"""World-size-2 gloo test of the multi-GPU host logic (sharding + one gather) on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_11462_b200.parallel import gather_results, rank_slice


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b0, b1 = rank_slice(12, world, rank)
    ids = np.arange(b0, b1)
    # stand-in per-rank translation results, a function of the global sentence index
    local = {"hyps": torch.tensor(np.stack([ids * 10 + j for j in range(4)], 1), dtype=torch.int32),
             "lens": torch.tensor(ids % 4 + 1, dtype=torch.int32),
             "scores": torch.tensor(-ids.astype(np.float32))}
    g = gather_results(local)
    q.put((rank, {k: v.numpy() for k, v in g.items()}))
    dist.destroy_process_group()


def test_rank_slices_partition_the_corpus():
    for world in (1, 2, 4, 8):
        cover = []
        for r in range(world):
            b0, b1 = rank_slice(240, world, r)
            cover += list(range(b0, b1))
        assert cover == list(range(240))
    with pytest.raises(ValueError):
        rank_slice(10, 2, 2)


def test_gloo_world2_gather_restores_corpus_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    ids = np.arange(12)
    for r in (0, 1):
        np.testing.assert_array_equal(res[r]["hyps"], np.stack([ids * 10 + j for j in range(4)], 1))
        np.testing.assert_array_equal(res[r]["lens"], ids % 4 + 1)
        np.testing.assert_array_equal(res[r]["scores"], -ids.astype(np.float32))
