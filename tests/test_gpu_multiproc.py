"""Two processes run the real CUDA path (one model handle each, on the one GPU this run has),
deal a corpus's batches round-robin, gather every output over gloo, and must reproduce the
one-process translation of the same batches BITWISE (fixed batch composition
makes the result independent of the process count).  The two ranks use the GPU one after the
other (a barrier), never concurrently: no kernel of one rank waits on the other."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu

N_SENT, BATCH, K, ML = 22, 6, 5, 12          # 4 batches, the last one ragged


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import paper_1805_11462_b200 as ob
    from paper_1805_11462_b200.parallel import deal_batches, gather_results, make_batches, translate_batches
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids, lens = synth.make_corpus("c2", N_SENT)
    batches = make_batches(N_SENT, BATCH)
    for r in range(world):                    # ranks take the GPU in turn
        if r == rank:
            with ob.Model(path, 0, "bf16") as m:
                local, idx = translate_batches(m, ids, lens, batches, deal_batches(len(batches), world, rank), K, ML)
        dist.barrier()
    g = gather_results({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in local.items()},
                       torch.from_numpy(idx), n_total=N_SENT)
    q.put((rank, {k: v.numpy() for k, v in g.items()}))
    dist.destroy_process_group()


def test_two_processes_equal_one_process_bitwise(weight_cache):
    import paper_1805_11462_b200 as ob
    from paper_1805_11462_b200.parallel import RESULT_KEYS, make_batches, translate_batches
    path = synth.weights_file("c2", weight_cache)
    ids, lens = synth.make_corpus("c2", N_SENT)
    with ob.Model(path, 0, "bf16") as m:
        one, idx = translate_batches(m, ids, lens, make_batches(N_SENT, BATCH), range(4), K, ML)
    assert list(idx) == list(range(N_SENT))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, path, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in (0, 1):
        for k in RESULT_KEYS:
            assert np.array_equal(res[r][k], one[k]), (r, k)
