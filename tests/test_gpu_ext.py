"""GPU parity of the translation customisations (onmt_translate_ex):
GNMT coverage penalty in the final score, n-best lists and attention-based unknown
replacement, against the fp64 oracle (oracle/beam.py beam_search(beta, n_best),
replace_unknowns)."""
import numpy as np
import pytest

import synth
from oracle import beam_search, replace_unknowns
from test_gpu_parity import model_pair, toy_pair

pytestmark = pytest.mark.gpu


def _src(ids, lens, b):
    return [int(v) for v in ids[b, :lens[b]]]


def test_ex_defaults_equal_translate(weight_cache):
    """beta = 0, n_best = 1, no replacement: bit-identical to onmt_translate."""
    for wl in ("c1",):
        gm, om, prec = model_pair(wl, weight_cache)
        ids, lens = synth.make_corpus(wl)
        a = gm.translate(ids, lens, 3, 10, 0.0)
        b = gm.translate_ex(ids, lens, 3, 10, 0.0)
        assert np.array_equal(a["hyps"], b["hyps"][:, 0]) and np.array_equal(a["lens"], b["lens"][:, 0])
        assert np.array_equal(a["scores"], b["scores"][:, 0]) and np.array_equal(a["token_logp"], b["token_logp"][:, 0])
    cfg = synth.ModelConfig(2, 64, 128, 300, 2000, False, True)
    gm, om, prec = toy_pair(cfg, 1, 0.1, weight_cache, "bf16")
    ids, lens = synth.make_corpus("c1")
    a = gm.translate(ids, lens, 5, 8, 0.6)
    b = gm.translate_ex(ids, lens, 5, 8, 0.6)
    assert np.array_equal(a["hyps"], b["hyps"][:, 0]) and np.array_equal(a["scores"], b["scores"][:, 0])


@pytest.mark.parametrize("alpha,beta,n_best", [(0.0, 0.2, 3), (0.6, 1.0, 3), (0.0, 0.0, 2), (1.0, 0.5, 1)])
def test_c1_fp32_coverage_nbest(weight_cache, alpha, beta, n_best):
    """c1 (fp32 mode): every n-best entry equals the oracle's - tokens exactly, final
    score (raw / lp + cp) and token log p within the fp32 bars."""
    gm, om, prec = model_pair("c1", weight_cache)
    ids, lens = synth.make_corpus("c1")
    K, ML = 3, 10
    out = gm.translate_ex(ids, lens, K, ML, alpha, beta, n_best)
    for b in range(len(lens)):
        ref = beam_search(om, _src(ids, lens, b), K, ML, alpha, beta=beta, n_best=n_best)
        assert len(ref["nbest"]) == n_best
        for i, e in enumerate(ref["nbest"]):
            n = out["lens"][b, i]
            assert list(out["hyps"][b, i, :n]) == e["tokens"], (b, i)
            assert abs(out["scores"][b, i] - e["norm"]) <= 1e-4 * max(1.0, abs(e["norm"]))
            assert abs(out["raw"][b, i] - e["raw"]) <= 1e-4 * max(1.0, abs(e["raw"]))
            np.testing.assert_allclose(out["token_logp"][b, i, :n], e["token_logp"], atol=1e-5)


@pytest.mark.parametrize("K,n_best,beta", [(5, 5, 0.4), (4, 2, 1.0)])
def test_peaky_bf16_coverage_nbest(weight_cache, K, n_best, beta):
    """bf16 toy model with EOS banked at every step (many bank entries): n-best lists
    match the oracle's (ranks whose final scores are within 1e-4 of a neighbour are
    tie-excused), scores within the bf16 bar."""
    cfg = synth.ModelConfig(2, 32, 64, 100, 40, False, True)
    gm, om, prec = toy_pair(cfg, 5, 0.3, weight_cache, "bf16", peaky=2.9, name="peaky_ext")
    ids, lens = synth.make_corpus("c1")
    ML = 8
    out = gm.translate_ex(ids, lens, K, ML, 0.6, beta, n_best)
    for b in range(len(lens)):
        ref = beam_search(om, _src(ids, lens, b), K, ML, 0.6, beta=beta, n_best=n_best)
        norms = [e["norm"] for e in ref["nbest"]]
        for i, e in enumerate(ref["nbest"]):
            n = out["lens"][b, i]
            tied = any(abs(norms[j] - e["norm"]) < 1e-4 for j in range(len(norms)) if j != i)
            if not tied:
                assert list(out["hyps"][b, i, :n]) == e["tokens"], (b, i)
            assert abs(out["scores"][b, i] - e["norm"]) <= 2e-3 * max(1, n)


def test_forced_unk_replacement(weight_cache):
    """Generator forced to <unk>, uniform attention (W_in = 0): every token is <unk> and
    is replaced by source position 0 (ties -> smallest s, S448)."""
    cfg = synth.ModelConfig(1, 32, 64, 100, 100, False, True)
    t = synth.random_model_tensors(cfg, 3, 0.1)
    ov = {"attn.w_in": np.zeros_like(t["attn.w_in"]), "gen.w": np.zeros_like(t["gen.w"]),
          "gen.b": np.where(np.arange(100) == 1, 50.0, 0.0).astype(np.float32)}
    for prec in ("fp32", "bf16"):
        gm, om, _ = toy_pair(cfg, 3, 0.1, weight_cache, prec, overrides=ov, name="forced_unk")
        ids, lens = synth.make_corpus("c1")
        out = gm.translate_ex(ids, lens, 3, 6, 0.0, 0.0, 1, True)
        assert (out["hyps"][:, 0] == 1).all()
        assert (out["unk_pos"][:, 0] == 0).all()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_unk_replacement_vs_oracle(weight_cache, prec):
    """A model that emits <unk> often (b[<unk>] raised): the replacement positions equal
    the oracle's attention argmax for every <unk> of the returned hypothesis."""
    cfg = synth.ModelConfig(2, 32, 64, 100, 200, prec == "bf16", True)
    t = synth.random_model_tensors(cfg, 11, 0.4)
    b = t["gen.b"].copy()
    b[1] = 2.5
    gm, om, _ = toy_pair(cfg, 11, 0.4, weight_cache, prec, overrides={"gen.b": b}, name="unk_often")
    ids, lens = synth.make_corpus("c1")
    out = gm.translate_ex(ids, lens, 3, 10, 0.0, 0.3, 2, True)
    n_unk = 0
    for bb in range(len(lens)):
        ref = beam_search(om, _src(ids, lens, bb), 3, 10, 0.0, beta=0.3, n_best=2)
        for i, e in enumerate(ref["nbest"]):
            n = out["lens"][bb, i]
            if list(out["hyps"][bb, i, :n]) != e["tokens"]:
                continue                                # (a near-tie divergence: nothing to compare)
            exp = replace_unknowns(e["tokens"], e["attn_argmax"])
            assert list(out["unk_pos"][bb, i, :n]) == exp
            assert (out["unk_pos"][bb, i, n:] == -1).all()
            n_unk += sum(1 for w in e["tokens"] if w == 1)
    assert n_unk > 0


def test_ex_errors(weight_cache):
    import paper_1805_11462_b200 as ob
    gm, om, prec = model_pair("c1", weight_cache)
    ids, lens = synth.make_corpus("c1")
    with pytest.raises(ob.OnmtError):
        gm.translate_ex(ids, lens, 3, 10, 0.0, 0.0, 4)      # n_best > beam
    with pytest.raises(ob.OnmtError):
        gm.translate_ex(ids, lens, 3, 10, 0.0, -1.0, 1)     # beta < 0


@pytest.mark.parametrize("layers,bidir", [(3, False), (2, False), (2, True)])
def test_persistent_encoders_match_per_step_path(weight_cache, layers, bidir):
    """The persistent encoders (enc_rec.cu; the unidirectional layer wavefront enc_wave.cu)
    compute the same memory bank and final states as the per-step launches, and both agree
    with the fp64 oracle."""
    cfg = synth.ModelConfig(layers, 64, 128, 300, 500, bidir, True)
    gm, om, prec = toy_pair(cfg, 21, 0.2, weight_cache, "bf16", name=f"enc{layers}{bidir}")
    ids, lens = synth.make_corpus("c1")
    ids = ids % 300
    ids[ids < 4] += 4
    mem1, h1, c1 = gm.encode(ids, lens)
    gm.set_option("enc_persistent", 0)
    try:
        mem0, h0, c0 = gm.encode(ids, lens)
    finally:
        gm.set_option("enc_persistent", 1)
    np.testing.assert_allclose(mem1, mem0, atol=5e-6)
    np.testing.assert_allclose(h1, h0, atol=5e-6)
    np.testing.assert_allclose(c1, c0, atol=5e-6)
    if bidir:                     # the cluster recurrence (enc_cl.cu) against the split-K grid kernel (enc_rec.cu)
        gm.set_option("enc_cluster", 0)
        try:
            mem2, h2, c2 = gm.encode(ids, lens)
        finally:
            gm.set_option("enc_cluster", 1)
        np.testing.assert_allclose(mem1, mem2, atol=5e-6)
        np.testing.assert_allclose(h1, h2, atol=5e-6)
        np.testing.assert_allclose(c1, c2, atol=5e-6)
    for b in range(len(lens)):
        ref_mem, finals = om.encode([int(v) for v in ids[b, :lens[b]]])
        np.testing.assert_allclose(mem1[b, :lens[b]], ref_mem, atol=2e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("h_dir", [128, 192, 320, 384, 448])
def test_cluster_encoder_widths(weight_cache, h_dir):
    """The cluster recurrence (enc_cl.cu) issues each step's MMAs as straight-line code per
    K-block count (h_dir / 64 = 2, 3, 5, 6, 7 here; 1 and 4 are covered above and by c3 / c5):
    it matches the split-K grid kernel and the fp64 oracle at every width.  (The two kernels sum
    the gate pre-activations in different fp32 orders - one accumulator per step against split-K
    partials - so at h_dir up to 448 they agree to ~1e-5, not bitwise; both are held to the
    oracle's 2e-4 bar.)"""
    cfg = synth.ModelConfig(2, 64, 2 * h_dir, 300, 500, True, True)
    gm, om, prec = toy_pair(cfg, 23, 0.2, weight_cache, "bf16", name=f"encw{h_dir}")
    ids, lens = synth.make_corpus("c1")
    ids = ids % 300
    ids[ids < 4] += 4
    mem1, h1, c1 = gm.encode(ids, lens)
    gm.set_option("enc_cluster", 0)
    try:
        mem2, h2, c2 = gm.encode(ids, lens)
    finally:
        gm.set_option("enc_cluster", 1)
    np.testing.assert_allclose(mem1, mem2, atol=2e-5)
    np.testing.assert_allclose(h1, h2, atol=2e-5)
    np.testing.assert_allclose(c1, c2, atol=2e-5)
    for b in range(0, len(lens), 3):
        ref_mem, finals = om.encode([int(v) for v in ids[b, :lens[b]]])
        np.testing.assert_allclose(mem1[b, :lens[b]], ref_mem, atol=2e-4)
