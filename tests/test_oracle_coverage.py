"""Pins for the oracle's coverage penalty, n-best lists and attention-based unknown
replacement (PAPER.md P313-316; SPEC.md S422-448).  CPU only.

Each pin is independent of the oracle's own arithmetic: SPEC worked examples, a
closed form under uniform attention (W_in = 0), brute-force enumeration at full beam
width, and a forced-output model."""
import math

import numpy as np
import pytest

import synth
from oracle import (OracleModel, beam_search, brute_force, coverage_penalty, final_score,
                    replace_unknowns)
from test_oracle_beam import TINY_V5_BI, TINY_V6, golden, toy


def test_coverage_golden():
    assert coverage_penalty(np.array([1.0, 2.5, 1.0]), 1.0) == golden("cp_beta1_all_covered")[0]
    assert abs(coverage_penalty(np.array([0.5, 2.0, 0.25]), 0.2) - golden("cp_beta02_hand")[0]) <= 1e-15
    assert coverage_penalty(np.array([0.1, 0.2]), 0.0) == 0.0          # S442: beta = 0 -> no penalty
    assert final_score(-3.0, 7, np.array([0.5]), 1.0, 0.0) == -1.5     # S443: lp(7) = 2 at alpha = 1


def test_replace_unknowns_golden():
    assert replace_unknowns([5, 1, 7, 1], [2, 0, 3, 1]) == [int(v) for v in golden("unk_replace_hand")]
    assert replace_unknowns([4, 5, 3], [1, 1, 0]) == [-1, -1, -1]      # S451: no <unk> -> unchanged


def _uniform_attention_model(cfg, seed, scale):
    """'general' attention with W_in = 0: every score is 0, so a_t = 1/S_b exactly."""
    t = {k: v.astype(np.float64) for k, v in synth.random_model_tensors(cfg, seed, scale).items()}
    t["attn.w_in"] = np.zeros_like(t["attn.w_in"])
    return OracleModel(t)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("beta", [0.2, 1.0])
def test_coverage_closed_form_uniform_attention(seed, beta):
    """Uniform attention: after n tokens every source position holds n/S_b, so
    cp = beta * S_b * log(min(n / S_b, 1)) for every banked hypothesis."""
    cfg = synth.ModelConfig(1, 4, 6, 12, 9, False, True)
    m = _uniform_attention_model(cfg, seed, 2.0)
    S = 3 + seed % 4
    src = list(np.random.default_rng(seed).integers(4, 12, S))
    out = beam_search(m, src, 4, 6, 0.0, beta=beta, n_best=4)
    for e in out["nbest"]:
        n = len(e["tokens"])
        expect = beta * S * math.log(min(n / S, 1.0))
        assert abs(e["cp"] - expect) <= 1e-12
        assert abs(e["norm"] - (e["raw"] + expect)) <= 1e-12


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("alpha,beta", [(0.0, 0.0), (0.0, 0.5), (0.6, 0.3), (1.0, 1.0)])
def test_full_width_nbest_equals_brute_force(seed, alpha, beta):
    """K >= V^max_len with no early stop: every sequence of Y is banked, so the n-best
    list is the top-n of the enumeration under final_score (S434 generalised to n-best,
    S436-439)."""
    cfg = TINY_V6 if seed % 2 == 0 else TINY_V5_BI
    m = toy(cfg, 300 + seed, 2.5)
    max_len = 3
    K = cfg.v_tgt ** max_len
    src = list(np.random.default_rng(seed).integers(4, 8, 1 + seed % 4))
    bf = brute_force(m, src, max_len, alpha, beta)
    n = 5
    b = beam_search(m, src, K, max_len, alpha, stop="none", beta=beta, n_best=n)
    got = [e["norm"] for e in b["nbest"]]
    np.testing.assert_allclose(got, [d["norm"] for d in bf[:n]], rtol=0, atol=1e-12)
    for i, e in enumerate(b["nbest"]):
        tied = any(abs(bf[j]["norm"] - bf[i]["norm"]) <= 1e-12 for j in range(len(bf)) if j != i)
        if not tied:
            assert e["tokens"] == bf[i]["tokens"]


@pytest.mark.parametrize("seed", range(8))
def test_nbest_order_and_prefix(seed):
    """n-best entries are in final order (norm desc, then step, then rank - AMB-19) and
    the first equals the single best."""
    cfg = synth.ModelConfig(2, 4, 6, 10, 12, seed % 2 == 1, True)
    m = toy(cfg, 40 + seed, 3.0)
    src = list(np.random.default_rng(seed).integers(4, 10, 4))
    out = beam_search(m, src, 5, 6, 0.6, beta=0.4, n_best=5)
    keys = [(-e["norm"], e["t"], e["r"]) for e in out["nbest"]]
    assert keys == sorted(keys)
    assert out["nbest"][0]["tokens"] == out["tokens"]
    with pytest.raises(ValueError):
        beam_search(m, src, 3, 6, n_best=4)                  # S423: n_best <= beam


def test_forced_unknown_replacement():
    """Generator forced to <unk> (W_gen = 0, b[<unk>] = +50) and uniform attention:
    every token is <unk> and is replaced by source position 0 (ties -> smallest s)."""
    cfg = synth.ModelConfig(1, 4, 6, 12, 9, False, True)
    t = {k: v.astype(np.float64) for k, v in synth.random_model_tensors(cfg, 3, 1.0).items()}
    t["attn.w_in"] = np.zeros_like(t["attn.w_in"])
    t["gen.w"] = np.zeros_like(t["gen.w"])
    t["gen.b"] = np.zeros_like(t["gen.b"])
    t["gen.b"][1] = 50.0
    m = OracleModel(t)
    out = beam_search(m, [5, 6, 7], 3, 5, 0.0)
    assert out["tokens"] == [1] * 5
    assert replace_unknowns(out["tokens"], out["attn_argmax"]) == [0] * 5
