"""World-size-2 gloo tests of the multi-GPU host logic on CPU: sharding with a
remainder, corpus batches dealt round-robin, and the one gather of every output plus the
original sentence indices restoring corpus order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_11462_b200.parallel import (RESULT_KEYS, deal_batches, gather_results, make_batches, rank_slice,
                                            translate_batches)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeModel:
    """CPU stand-in with the binding's translate() signature: every output is a function of
    the sentence's own ids (so any mix-up of rows shows), independent of the batch."""

    def translate(self, ids, lens, beam, max_len, alpha):
        B = len(lens)
        key = (ids.astype(np.int64) * np.arange(1, ids.shape[1] + 1)).sum(1) + lens
        hyps = (key[:, None] + np.arange(max_len)[None]).astype(np.int32) % 997
        return {"hyps": hyps, "lens": (key % max_len + 1).astype(np.int32),
                "scores": (-key / 7.0).astype(np.float32), "raw": (-key / 3.0).astype(np.float32),
                "token_logp": np.tile((-key / 11.0).astype(np.float32)[:, None], (1, max_len))[:B]}


def _corpus(n):
    rng = np.random.default_rng(3)
    lens = rng.integers(1, 9, n).astype(np.int32)
    ids = np.zeros((n, 8), np.int32)
    for b in range(n):
        ids[b, :lens[b]] = rng.integers(4, 50, lens[b])
    return ids, lens


def _worker(rank, world, port, q, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 23                                                     # not a multiple of the world size
    ids, lens = _corpus(n)
    m = FakeModel()
    if mode == "corpus":                                       # batches of 4, dealt round-robin
        batches = make_batches(n, 4)
        local, idx = translate_batches(m, ids, lens, batches, deal_batches(len(batches), world, rank), 3, 6)
    else:                                                      # one batch sharded by sentence
        b0, b1 = rank_slice(n, world, rank)
        local = m.translate(ids[b0:b1], lens[b0:b1], 3, 6, 0.0)
        idx = np.arange(b0, b1)
    g = gather_results({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in local.items()},
                       torch.from_numpy(idx), n_total=n)
    q.put((rank, {k: v.numpy() for k, v in g.items()}))
    dist.destroy_process_group()


def test_rank_slices_partition_the_corpus():
    for n in (240, 23, 7, 1, 0):
        for world in (1, 2, 3, 4, 8):
            cover, sizes = [], []
            for r in range(world):
                b0, b1 = rank_slice(n, world, r)
                cover += list(range(b0, b1))
                sizes.append(b1 - b0)
            assert cover == list(range(n))                     # nothing dropped, nothing twice
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        rank_slice(10, 2, 2)


def test_round_robin_deal_covers_every_batch():
    batches = make_batches(3840, 30)
    assert len(batches) == 128 and batches[-1] == (3810, 3840)
    assert make_batches(23, 4)[-1] == (20, 23)
    for world in (1, 2, 4, 8, 3):
        dealt = sorted(i for r in range(world) for i in deal_batches(len(batches), world, r))
        assert dealt == list(range(len(batches)))


@pytest.mark.parametrize("mode", ["corpus", "shard"])
def test_gloo_world2_gather_restores_corpus_order(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    ids, lens = _corpus(23)
    want = FakeModel().translate(ids, lens, 3, 6, 0.0)         # one process, whole corpus
    for r in (0, 1):
        for k in RESULT_KEYS:
            np.testing.assert_array_equal(res[r][k], want[k])


class FakeVpModel:
    """Records the vocabulary-parallel set-up calls (the handle bytes identify the rank)."""

    def __init__(self, rank):
        self.rank = rank
        self.opened = None

    def vp_handle(self, max_rows):
        return bytes([self.rank]) * 32 + max_rows.to_bytes(32, "little")

    def vp_open(self, world, rank, handles):
        self.opened = (world, rank, handles)


def _vp_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_11462_b200.parallel import open_vocab_parallel
    m = FakeVpModel(rank)
    open_vocab_parallel(m, 150)
    q.put((rank, m.opened))
    dist.destroy_process_group()


def test_gloo_world2_vocab_parallel_handle_exchange():
    """Every rank maps every rank's exchange buffer: the handles arrive in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_vp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    want = b"".join(bytes([r]) * 32 + (150).to_bytes(32, "little") for r in range(2))
    for r in (0, 1):
        world, rank, handles = res[r]
        assert (world, rank) == (2, r) and handles == want
