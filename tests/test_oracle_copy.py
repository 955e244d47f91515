"""Pins for the oracle's copy / pointer generator (PAPER.md P302-304,
P316-317 "copy mechanism", "dynamic dictionary support for copy/pointer networks";
SPEC.md S293-301).  CPU only.  Independent checks: SPEC worked examples, a hand-computed
mixture, normalisation by direct summation, the g -> 1 limit, full-width beam search over
the extended vocabulary == brute-force enumeration, and the <unk> feed-back reading."""
import math

import numpy as np
import pytest

import synth
from oracle import OracleModel, beam_search, brute_force, score_sequence
from test_oracle_beam import golden


def copy_model(cfg, seed, scale, gate_bias=None):
    t = {k: v.astype(np.float64) for k, v in synth.random_model_tensors(cfg, seed, scale).items()}
    if gate_bias is not None:
        t["copy.w"] = np.zeros_like(t["copy.w"])
        t["copy.b"] = np.array([gate_bias])
    return OracleModel(t)


def test_extended_log_probs_golden():
    f = OracleModel.extended_log_probs
    lp = np.log(np.array([[0.1, 0.2, 0.3, 0.4]]))
    got = np.exp(f(lp, np.array([[0.5, 0.5]]), np.array([0.25]), [1, 4], 5))[0]
    np.testing.assert_allclose(got, golden("copy_mix_hand"), rtol=0, atol=1e-15)
    # S299: g = 0 and one-hot attention on position 1 -> all mass on src_ext[1]
    v = f(np.log(np.full((1, 8), 1 / 8)), np.array([[0.0, 1.0, 0.0]]), np.array([0.0]), [5, 7, 5], 8)[0]
    assert v[7] == golden("copy_g0_onehot")[0] and np.all(np.isneginf(np.delete(v, 7)))


CFG = synth.ModelConfig(1, 4, 6, 12, 7, False, True, copy=True)


@pytest.mark.parametrize("seed", range(6))
def test_extended_distribution_normalised(seed):
    """S300: the extended probabilities of a real step sum to 1 (direct summation)."""
    m = copy_model(CFG, seed, 1.5)
    src = list(np.random.default_rng(seed).integers(4, 12, 4))
    ext = [w if w < 7 and w % 2 == 0 else 7 + i for i, w in enumerate(src)]
    out = beam_search(m, src, 3, 4, src_ext=ext, trace=True)
    lp = score_sequence(m, src, out["tokens"], src_ext=ext)
    assert all(x <= 0 for x in lp)
    from oracle.beam import _step_log_probs
    mem, fin = m.encode(src)
    y, ht, st = m.init_decoder(fin, 1)
    logp, _, _, _ = _step_log_probs(m, y, ht, st, mem, ext)
    assert abs(np.exp(logp).sum() - 1.0) <= 1e-10


def test_gate_one_equals_generator():
    """S298: g = 1 -> the extended distribution is the generator's, zero on source-only ids."""
    m = copy_model(CFG, 2, 1.5, gate_bias=60.0)          # sigmoid(60) == 1.0 in fp64
    m0 = OracleModel({k: v for k, v in m.t.items() if not k.startswith("copy.")})
    src = [5, 9, 6, 11]
    ext = [5, 7, 6, 8]
    a = beam_search(m, src, 3, 5, src_ext=ext)
    b = beam_search(m0, src, 3, 5)
    assert a["tokens"] == b["tokens"]
    np.testing.assert_allclose(a["token_logp"], b["token_logp"], atol=1e-12)


@pytest.mark.parametrize("seed", range(12))
def test_full_width_copy_beam_equals_brute_force(seed):
    """K >= V_ext^max_len: beam search over the extended vocabulary keeps every candidate,
    so its best raw score is the exact argmax over all sequences of extended ids (S434)."""
    cfg = synth.ModelConfig(1, 3, 4, 8, 5, seed % 2 == 1, True, copy=True)
    m = copy_model(cfg, 50 + seed, 2.5)
    src = list(np.random.default_rng(seed).integers(4, 8, 2 + seed % 2))
    ext = [5 + i if i % 2 == 0 else min(w, 4) for i, w in enumerate(src)]   # two source-only ids
    v_ext = max(5, max(ext) + 1)
    max_len = 3
    bf = brute_force(m, src, max_len, src_ext=ext)
    b = beam_search(m, src, v_ext ** max_len, max_len, 0.0, stop="none", src_ext=ext)
    assert abs(b["raw"] - bf[0]["raw"]) <= 1e-12
    if abs(bf[0]["raw"] - bf[1]["raw"]) > 1e-12:
        assert b["tokens"] == bf[0]["tokens"]


def test_extended_id_fed_back_as_unk():
    """Reading R32: an emitted source-only id (>= V) is fed to the next step as <unk>, so the
    continuation's log-probs equal those after an emitted <unk>."""
    m = copy_model(CFG, 4, 1.5)
    src = [5, 9, 6]
    ext = [5, 7, 8]
    y1 = score_sequence(m, src, [4, 7, 6, 3], src_ext=ext)
    y2 = score_sequence(m, src, [4, 1, 6, 3], src_ext=ext)
    np.testing.assert_allclose(y1[2:], y2[2:], atol=1e-14)
    assert y1[1] != y2[1]


@pytest.mark.parametrize("seed", range(4))
def test_copy_gate_reads_attentional_vector(seed):
    """copy_gate with w != 0 (reading R31: g = sigmoid(copy.w . h~ + copy.b), h~ the attentional
    vector, SPEC S293-297).  Closed-form model: W_in = 0 (uniform attention a_s = 1/S, S273-style),
    W_out = [0 | kappa I] (h~ = tanh(kappa h_1)), W_gen = 0, b_gen = 0 (p_vocab = 1/V), so
    p(w) = g / V + (1 - g) n_w / S (S296).  h_1 comes from torch.nn.LSTM / LSTMCell (library),
    not from the oracle; feeding h_1 instead of h~ to the gate, a wrong sign or a dropped bias
    fails it."""
    import torch
    cfg = synth.ModelConfig(1, 5, 6, 12, 9, False, True, copy=True)
    t = {k: v.astype(np.float64) for k, v in synth.random_model_tensors(cfg, 70 + seed, 1.0).items()}
    H, V, kappa = 6, 9, 2.0
    t["attn.w_in"] = np.zeros((H, H))
    t["attn.w_out"] = np.concatenate([np.zeros((H, H)), kappa * np.eye(H)], axis=1)
    t["gen.w"] = np.zeros((V, H))
    t["gen.b"] = np.zeros(V)
    rng = np.random.default_rng(seed)
    t["copy.w"] = rng.uniform(-2, 2, (1, H))
    t["copy.b"] = np.array([rng.uniform(-1, 1)])
    m = OracleModel(t)
    src = [5, 9, 5, 11]
    ext = [5, 9 + 0, 5, 10]                 # id 5 shared twice, 9 and 10 source-only (V = 9)
    with torch.no_grad():
        enc = torch.nn.LSTM(5, H, 1, batch_first=True).double()
        enc.weight_ih_l0.copy_(torch.from_numpy(t["enc.l0.fwd.w_ih"]))
        enc.weight_hh_l0.copy_(torch.from_numpy(t["enc.l0.fwd.w_hh"]))
        enc.bias_ih_l0.copy_(torch.from_numpy(t["enc.l0.fwd.b_ih"]))
        enc.bias_hh_l0.copy_(torch.from_numpy(t["enc.l0.fwd.b_hh"]))
        x = torch.from_numpy(t["enc.emb"][src])[None]
        _, (h0, c0) = enc(x)
        cell = torch.nn.LSTMCell(5 + H, H).double()
        cell.weight_ih.copy_(torch.from_numpy(t["dec.l0.w_ih"]))
        cell.weight_hh.copy_(torch.from_numpy(t["dec.l0.w_hh"]))
        cell.bias_ih.copy_(torch.from_numpy(t["dec.l0.b_ih"]))
        cell.bias_hh.copy_(torch.from_numpy(t["dec.l0.b_hh"]))
        u = torch.cat([torch.from_numpy(t["dec.emb"][2]), torch.zeros(H, dtype=torch.float64)])[None]
        h1, _ = cell(u, (h0[0], c0[0]))
        ht = torch.tanh(kappa * h1[0]).numpy()
    g = 1.0 / (1.0 + math.exp(-(float(t["copy.w"][0] @ ht) + float(t["copy.b"][0]))))
    S = len(src)
    want = {5: g / V + (1 - g) * 2 / S, 9: (1 - g) / S, 10: (1 - g) / S, 4: g / V}
    for w, p in want.items():
        got = score_sequence(m, src, [w], src_ext=ext)[0]
        assert abs(got - math.log(p)) <= 1e-12, (w, got, math.log(p))
