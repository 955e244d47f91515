"""Teacher-forced scoring (onmt_score) against the fp64 oracle's
score_sequence (PAPER.md P105-108), through the C-ABI."""
import numpy as np
import pytest

import synth
from oracle import score_sequence

pytestmark = pytest.mark.gpu

from test_gpu_parity import model_pair  # noqa: E402  (same model cache)


def random_targets(V, B, T_max, seed, lo=1):
    rng = np.random.default_rng(seed)
    tlens = rng.integers(lo, T_max + 1, B).astype(np.int32)
    tgt = np.zeros((B, T_max), np.int32)
    for b in range(B):
        tgt[b, :tlens[b]] = rng.integers(4, V, tlens[b])
        if rng.random() < 0.5:
            tgt[b, tlens[b] - 1] = synth.EOS
    return tgt, tlens


def check(gm, om, ids, lens, tgt, tlens, tol):
    out = gm.score(ids, lens, tgt, tlens)
    for b in range(len(lens)):
        ref = score_sequence(om, [int(v) for v in ids[b, :lens[b]]], [int(v) for v in tgt[b, :tlens[b]]])
        got = out["token_logp"][b, :tlens[b]]
        np.testing.assert_allclose(got, ref, atol=tol, rtol=0)
        assert (out["token_logp"][b, tlens[b]:] == 0).all()
        np.testing.assert_allclose(out["nll"][b], -np.sum(ref), atol=tol * tlens[b])


def test_score_c1_fp32(weight_cache):
    gm, om, p = model_pair("c1", weight_cache)
    ids, lens = synth.make_corpus("c1")
    tgt, tlens = random_targets(100, len(lens), 12, 0)
    check(gm, om, ids, lens, tgt, tlens, 1e-5)


@pytest.mark.parametrize("workload,n", [("c2", 6), ("c3", 4)])
def test_score_bf16(workload, n, weight_cache):
    gm, om, p = model_pair(workload, weight_cache)
    ids, lens = synth.make_corpus(workload, n)
    tgt, tlens = random_targets(50000, len(lens), 9, 1)
    check(gm, om, ids, lens, tgt, tlens, 2e-3)


def test_score_matches_translation_logp(weight_cache):
    """Scoring the beam's own 1-best reproduces the per-token log-probs the beam reported."""
    gm, om, p = model_pair("c2", weight_cache)
    ids, lens = synth.make_corpus("c2", 5)
    tr = gm.translate(ids, lens, 5, 10, 0.0)
    sc = gm.score(ids, lens, tr["hyps"], tr["lens"])
    for b in range(len(lens)):
        n = tr["lens"][b]
        np.testing.assert_allclose(sc["token_logp"][b, :n], tr["token_logp"][b, :n], atol=1e-4)


def test_score_errors(weight_cache):
    import paper_1805_11462_b200 as ob
    gm, om, p = model_pair("c1", weight_cache)
    ids, lens = synth.make_corpus("c1")
    tgt, tlens = random_targets(100, len(lens), 5, 2)
    with pytest.raises(ob.OnmtError) as e:
        gm.score(ids, lens, tgt, np.zeros_like(tlens))
    assert e.value.name == "EMPTY_SOURCE"
    bad = tgt.copy()
    bad[0, 0] = 100
    with pytest.raises(ob.OnmtError) as e:
        gm.score(ids, lens, bad, tlens)
    assert e.value.name == "ID_RANGE"
    # T_max = 1, single-token targets
    one = gm.score(ids, lens, tgt[:, :1], np.ones(len(lens), np.int32))
    assert one["token_logp"].shape == (len(lens), 1)
