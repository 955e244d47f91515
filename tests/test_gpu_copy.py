"""GPU parity of the copy / pointer generator (onmt_translate_copy):
beam search over the extended vocabulary against the fp64 oracle (oracle/beam.py
beam_search(src_ext) / score_sequence(src_ext))."""
import os

import numpy as np
import pytest

import synth
from oracle import OracleModel, beam_search, load_model_tensors, score_sequence

pytestmark = pytest.mark.gpu


def _pair(weight_cache, cfg, seed, scale, prec, gate_bias=None, name="copy"):
    import paper_1805_11462_b200 as ob
    t = synth.random_model_tensors(cfg, seed, scale)
    if gate_bias is not None:
        t["copy.b"] = np.array([gate_bias], np.float32)
    path = os.path.join(weight_cache, f"{name}_{seed}_{prec}_{abs(hash(str(cfg))) % 10**8}.mnmt")
    synth.write_mnmt(path, t)
    return ob.Model(path, 0, prec), OracleModel(load_model_tensors(path, prec))


def _src(a, lens, b):
    return [int(v) for v in a[b, :lens[b]]]


@pytest.mark.parametrize("gate_bias", [None, -2.0])
def test_copy_fp32_exact(weight_cache, gate_bias):
    """fp32 mode: the same hypotheses as the oracle, token log p within 1e-5."""
    cfg = synth.ModelConfig(1, 32, 64, 100, 100, False, True, copy=True)
    gm, om = _pair(weight_cache, cfg, 7, 0.3, "fp32", gate_bias)
    ids, lens = synth.make_corpus("c1")
    ext = synth.make_src_ext(ids, lens, 100)
    out = gm.translate_copy(ids, lens, ext, 3, 10, 0.0)
    n_ext = 0
    for b in range(len(lens)):
        ref = beam_search(om, _src(ids, lens, b), 3, 10, 0.0, src_ext=_src(ext, lens, b))
        n = out["lens"][b]
        assert list(out["hyps"][b, :n]) == ref["tokens"], b
        np.testing.assert_allclose(out["token_logp"][b, :n], ref["token_logp"], atol=1e-5)
        assert abs(out["scores"][b] - ref["norm"]) <= 1e-4
        n_ext += sum(1 for w in ref["tokens"] if w >= 100)
    if gate_bias is not None:
        assert n_ext > 0                                 # copied source-only words were emitted


@pytest.mark.parametrize("bidir", [False, True])
def test_copy_bf16_teacher_forced(weight_cache, bidir):
    """bf16 mode: the GPU's own hypotheses scored by teacher forcing in the oracle agree
    token by token within 2e-3 (R21), and the raw score equals their sum."""
    cfg = synth.ModelConfig(2, 64, 128, 300, 2000, bidir, True, copy=True)
    gm, om = _pair(weight_cache, cfg, 9, 0.1, "bf16", -1.0)
    ids, lens = synth.make_corpus("c1")
    ids = ids % 300
    ids[ids < 4] += 4
    ext = synth.make_src_ext(ids, lens, 2000)
    out = gm.translate_copy(ids, lens, ext, 5, 8, 0.0)
    for b in range(len(lens)):
        n = out["lens"][b]
        hyp = [int(v) for v in out["hyps"][b, :n]]
        ref = score_sequence(om, _src(ids, lens, b), hyp, src_ext=_src(ext, lens, b))
        np.testing.assert_allclose(out["token_logp"][b, :n], ref, atol=2e-3)
        assert abs(out["raw"][b] - float(np.sum(out["token_logp"][b, :n]))) <= 1e-3


def test_copy_errors(weight_cache):
    import paper_1805_11462_b200 as ob
    cfg = synth.ModelConfig(1, 32, 64, 100, 100, False, True, copy=True)
    gm, om = _pair(weight_cache, cfg, 7, 0.3, "fp32")
    ids, lens = synth.make_corpus("c1")
    with pytest.raises(ob.OnmtError):
        gm.translate(ids, lens, 3, 10)                   # a copy model needs src_ext
    bad = synth.make_src_ext(ids, lens, 100)
    bad[0, 0] = 100 + ids.shape[1]                       # outside [0, V + S_max)
    with pytest.raises(ob.OnmtError):
        gm.translate_copy(ids, lens, bad, 3, 10)
    cfg2 = synth.ModelConfig(1, 32, 64, 100, 100, False, True)
    gm2, _ = _pair(weight_cache, cfg2, 7, 0.3, "fp32", name="nocopy")
    with pytest.raises(ob.OnmtError):
        gm2.translate_copy(ids, lens, synth.make_src_ext(ids, lens, 100), 3, 10)
