"""Vocabulary-parallel generator on the one GPU this run has.

A world of 1 runs the whole protocol - the generator stores its partials through the peer-pointer
array into the (own) exchange buffer and raises its per-step flags, the beam step waits for every
flag of the step epoch and merges the exchanged partials - and must return exactly the single-GPU
translation (same CTA split, same merge order).  Worlds > 1 need one GPU per rank (no kernel may
wait on another rank's kernel on a shared GPU); they are unmeasured in this run."""
import numpy as np
import pytest

import synth
from parity import compare_batch
from test_gpu_parity import model_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workload,n,max_len", [("c2", 30, 24), ("c5", 16, 12)])
def test_world1_equals_single_gpu_bitwise(workload, n, max_len, weight_cache):
    gm, om, prec = model_pair(workload, weight_cache)
    w = synth.WORKLOADS[workload]
    ids, lens = synth.make_corpus(workload, n)
    K, alpha = w.decode.beam, w.decode.alpha
    gm.set_option("rsplit", 0)                       # (vocabulary-parallel decoding runs the per-layer step)
    try:
        ref = gm.translate(ids, lens, K, max_len, alpha)
        gm.vp_handle(n * K)
        gm.vp_open(1, 0, None)
        try:
            a = gm.translate(ids, lens, K, max_len, alpha)
            b = gm.translate(ids, lens, K, max_len, alpha, trace=True)     # a second call: new flag epochs
            plan = gm.last_plan()
        finally:
            gm.vp_close()
    finally:
        gm.set_option("rsplit", 1)
    assert plan["rsplit"] == 0
    for k in ("hyps", "lens", "scores", "raw", "token_logp"):
        assert np.array_equal(a[k], ref[k]), k
        assert np.array_equal(b[k], ref[k]), k
    res = compare_batch(om, ids, lens, b, K, max_len, alpha, prec, sentences=[0, n - 1])
    assert res["fail"] == 0, res["details"]


def test_vp_errors(weight_cache):
    import paper_1805_11462_b200 as ob
    gm, om, prec = model_pair("c2", weight_cache)
    with pytest.raises(ob.OnmtError):
        gm.vp_open(2, 2, None)                       # rank >= world
    gm.vp_handle(10)                                 # capacity: 10 rows
    gm.vp_open(1, 0, None)
    try:
        ids, lens = synth.make_corpus("c2", 4)
        with pytest.raises(ob.OnmtError) as e:
            gm.translate(ids, lens, 5, 4, 0.0)       # 20 rows > capacity
        assert e.value.name == "UNSUPPORTED"
    finally:
        gm.vp_close()
    out = gm.translate(ids, lens, 5, 4, 0.0)         # single-GPU decoding again
    assert out["lens"].shape == (4,)


@pytest.mark.parametrize("world", [2, 4])
def test_vocab_split_emulated_ranks_bitwise(world, weight_cache):
    """The vocabulary split itself: `world` ranks emulated by sequential generator launches on this
    GPU, rank r running CTAs [r C / world, (r + 1) C / world) of the C-CTA split and storing its
    partial columns through the exchange pointers; the merged LSE and top-K equal the one-launch
    generator's bitwise (same partials, same merge order)."""
    gm, om, prec = model_pair("c2", weight_cache)
    rng = np.random.default_rng(world)
    h = np.tanh(rng.normal(size=(150, 500))).astype(np.float32)
    ref = gm.test_gen(h, 5)
    gm.set_option("test_gen_world", world)
    try:
        got = gm.test_gen(h, 5)
    finally:
        gm.set_option("test_gen_world", 0)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)
