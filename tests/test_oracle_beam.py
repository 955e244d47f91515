"""Pins for the oracle's beam search (CPU only): greedy, brute force, closed forms
and invariants (BASELINE.json north_star's four oracle checks + SPEC extras)."""
import heapq
import itertools
import math
import os

import numpy as np
import pytest

import synth
from oracle import (OracleModel, beam_search, brute_force, greedy, length_penalty,
                    score_sequence, translate_batch)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    for line in open(os.path.join(GOLD, "worked_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        parts = [p.strip() for p in line.split("|")]
        if parts[0] == name:
            return [float(v) for v in parts[2].split(",")]
    raise KeyError(name)


def toy(cfg, seed, scale, overrides=None):
    t = {k: v.astype(np.float64) for k, v in synth.random_model_tensors(cfg, seed, scale).items()}
    if overrides:
        t.update(overrides)
    return OracleModel(t)


TINY_V6 = synth.ModelConfig(1, 3, 4, 8, 6, False, True)
TINY_V5_BI = synth.ModelConfig(2, 3, 4, 8, 5, True, False)


def test_length_penalty_golden():
    assert length_penalty(7, 1.0) == golden("lp_alpha1_len7")[0]
    assert length_penalty(7, 0.0) == golden("lp_alpha0_len7")[0]


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("alpha", [0.0, 0.6])
def test_beam1_equals_greedy(seed, alpha):
    cfg = synth.ModelConfig(2, 4, 6, 10, 9, seed % 2 == 1, seed % 3 != 0)
    m = toy(cfg, seed, 1.5)
    src = list(np.random.default_rng(seed).integers(4, 10, 1 + seed % 5))
    g = greedy(m, src, 7)
    b = beam_search(m, src, 1, 7, alpha)
    assert b["tokens"] == g["tokens"]
    np.testing.assert_allclose(b["token_logp"], g["token_logp"], atol=0)


@pytest.mark.parametrize("seed", range(40))
def test_full_width_beam_equals_brute_force(seed):
    """K >= V^max_len, alpha = 0: the beam keeps every candidate, so its best
    raw score is the exact argmax over all finite sequences (north_star check 1)."""
    cfg = TINY_V6 if seed % 2 == 0 else TINY_V5_BI
    m = toy(cfg, seed, 2.0 + seed % 3)          # peaky distributions so EOS wins sometimes
    max_len = 3
    K = cfg.v_tgt ** max_len
    src = list(np.random.default_rng(seed).integers(4, 8, 1 + seed % 4))
    bf = brute_force(m, src, max_len)
    b = beam_search(m, src, K, max_len, 0.0)
    assert abs(b["raw"] - bf[0]["raw"]) <= 1e-12
    if abs(bf[0]["raw"] - bf[1]["raw"]) > 1e-12:
        assert b["tokens"] == bf[0]["tokens"]


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("alpha", [0.6, 1.0])
def test_full_width_length_normalised_equals_brute_force(seed, alpha):
    cfg = TINY_V6 if seed % 2 == 0 else TINY_V5_BI
    m = toy(cfg, 100 + seed, 2.5)
    max_len = 3
    K = cfg.v_tgt ** max_len
    src = list(np.random.default_rng(seed).integers(4, 8, 2))
    bf = brute_force(m, src, max_len, alpha)
    for stop in ("none", "bound"):
        b = beam_search(m, src, K, max_len, alpha, stop=stop)
        assert abs(b["norm"] - bf[0]["norm"]) <= 1e-12, stop


def test_forced_model_eos():
    """W_gen = 0, b_gen[EOS] = 50: [EOS] with raw = -log(1 + (V-1) e^-50) (S435)."""
    cfg = synth.ModelConfig(1, 4, 6, 20, 20, False, True)
    b = np.zeros(20); b[synth.EOS] = 50.0
    m = toy(cfg, 0, 0.3, {"gen.w": np.zeros((20, 6)), "gen.b": b})
    r = beam_search(m, [4, 5, 6], 5, 10)
    assert r["tokens"] == [synth.EOS]
    # fp64 cannot resolve 19 e^-50 next to 50: raw is exact up to ulp(50)
    assert abs(r["raw"] - (-math.log1p(19 * math.exp(-50)))) < 8e-15
    b[synth.EOS] = 10.0                          # resolvable: raw = -log(1 + 19 e^-10)
    m = toy(cfg, 0, 0.3, {"gen.w": np.zeros((20, 6)), "gen.b": b})
    r = beam_search(m, [4, 5, 6], 5, 10)
    assert r["tokens"] == [synth.EOS]
    assert abs(r["raw"] - (-math.log1p(19 * math.exp(-10)))) < 1e-14


@pytest.mark.parametrize("K,max_len", [(3, 4), (7, 3), (1, 5)])
def test_unigram_model_kbest_by_enumeration(K, max_len):
    """W_out = 0 -> h~ = 0 -> log p = log_softmax(b) at every step; with EOS
    made impossible the beam's K slots at t = max_len are the exact K best sums
    of max_len unigram log-probs (enumerated independently)."""
    cfg = synth.ModelConfig(1, 3, 4, 9, 7, False, True)
    rng = np.random.default_rng(K)
    bias = rng.normal(size=7); bias[synth.EOS] = -60.0
    m = toy(cfg, 1, 0.5, {"attn.w_out": np.zeros((4, 8)), "gen.b": bias})
    u = bias - (bias.max() + math.log(np.exp(bias - bias.max()).sum()))
    sums = sorted((sum(u[w] for w in seq), seq) for seq in itertools.product(range(7), repeat=max_len))
    best = heapq.nlargest(K, [s for s, _ in sums])
    r = beam_search(m, [4, 5], K, max_len)
    final = [e for e in r["bank"] if e[1] == max_len]
    raws = sorted([e[3] for e in final], reverse=True)
    np.testing.assert_allclose(raws, best, atol=1e-12)
    # anything banked earlier is an EOS pick (score ~ -60, never among the K best)
    assert all(e[4][-1] == synth.EOS and e[3] < -50 for e in r["bank"] if e[1] < max_len)


@pytest.mark.parametrize("seed", range(6))
def test_score_bookkeeping_and_teacher_forcing(seed):
    cfg = synth.ModelConfig(2, 5, 6, 30, 25, seed % 2 == 0, seed % 2 == 1)
    m = toy(cfg, seed, 1.0)
    src = list(np.random.default_rng(seed).integers(4, 30, 6))
    r = beam_search(m, src, 4, 8, 0.5)
    assert abs(sum(r["token_logp"]) - r["raw"]) < 1e-12            # S476
    np.testing.assert_allclose(score_sequence(m, src, r["tokens"]), r["token_logp"], atol=1e-12)
    assert abs(r["norm"] - r["raw"] / length_penalty(len(r["tokens"]), 0.5)) < 1e-12


def test_batch_equivalence_and_permutation():
    cfg = synth.ModelConfig(2, 5, 6, 30, 25, False, True)
    m = toy(cfg, 3, 1.0)
    rng = np.random.default_rng(0)
    srcs = [list(rng.integers(4, 30, n)) for n in (3, 7, 1, 5)]
    batch = translate_batch(m, srcs, 3, 6)
    singles = [beam_search(m, s, 3, 6) for s in srcs]
    for a, b in zip(batch, singles):
        assert a["tokens"] == b["tokens"] and a["raw"] == b["raw"]
    perm = [2, 0, 3, 1]
    pb = translate_batch(m, [srcs[i] for i in perm], 3, 6)
    for j, i in enumerate(perm):
        assert pb[j]["tokens"] == batch[i]["tokens"] and pb[j]["raw"] == batch[i]["raw"]
    assert translate_batch(m, [], 3, 6) == []                        # S471


def test_random_weights_run_to_max_len():
    """with U(-0.1,0.1) weights EOS essentially never ranks first."""
    cfg = synth.ModelConfig(1, 16, 32, 200, 2000, False, True)
    m = toy(cfg, 0, 0.1)
    r = beam_search(m, [5, 9, 11, 40], 5, 12)
    assert r["t"] == 12 and len(r["tokens"]) == 12


def test_errors():
    m = toy(TINY_V6, 0, 1.0)
    with pytest.raises(ValueError):
        beam_search(m, [], 2, 3)
    with pytest.raises(ValueError):
        beam_search(m, [4], 0, 3)
