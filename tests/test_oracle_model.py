"""Pins for the oracle's model pieces (CPU only).  DESIGN.md §4 lists which pin
covers which function; none of them re-derives the oracle from itself."""
import math
import os
import struct

import numpy as np
import pytest
import scipy.special
import torch

import synth
from oracle import OracleModel, bf16_round, read_mnmt
from oracle.model import lstm_cell

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    for line in open(os.path.join(GOLD, "worked_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        parts = [p.strip() for p in line.split("|")]
        if parts[0] == name:
            return [float(v) for v in parts[2].split(",")]
    raise KeyError(name)


def toy_model(cfg, seed=0, scale=0.1, overrides=None):
    t = {k: v.astype(np.float64) for k, v in synth.random_model_tensors(cfg, seed, scale).items()}
    if overrides:
        t.update(overrides)
    return OracleModel(t)


SMALL = synth.ModelConfig(2, 6, 8, 13, 11, False, True)
SMALL_BI = synth.ModelConfig(2, 6, 8, 13, 11, True, False)


# ------------------------------------------------------------------ container / bf16
def test_mnmt_golden_bytes(tmp_path):
    hexline = [l for l in open(os.path.join(GOLD, "mnmt_tiny.hex")) if not l.startswith("#")][0].strip()
    p = tmp_path / "tiny.mnmt"
    p.write_bytes(bytes.fromhex(hexline))
    t = read_mnmt(str(p))
    assert list(t) == ["a", "b.c"]
    np.testing.assert_array_equal(t["a"], np.array([[1, -2, 0.5], [0.25, -0.125, 3]], np.float32))
    np.testing.assert_array_equal(t["b.c"], np.array([-1.5], np.float32))


def test_mnmt_roundtrip_synth_writer(tmp_path):
    w = synth.make_weights(SMALL, 3)
    p = str(tmp_path / "m.mnmt")
    synth.write_mnmt(p, w)
    r = read_mnmt(p)
    assert list(r) == [n for n, _ in synth.tensor_specs(SMALL)]
    for k in w:
        np.testing.assert_array_equal(r[k], w[k])


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-0.1, 0.1, 100000), rng.normal(0, 1e3, 1000),
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 0.0, -0.0])]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    np.testing.assert_array_equal(bf16_round(x), ref)
    # ties-to-even worked by hand: 1+2^-8 is halfway between 1 and 1+2^-7 -> 1
    assert bf16_round(np.array([1.0 + 2 ** -8], np.float32))[0] == 1.0
    assert bf16_round(np.array([1.0 + 3 * 2 ** -8], np.float32))[0] == 1.0 + 2 ** -6


# ------------------------------------------------------------------ LSTM cell / encoder
def test_lstm_cell_matches_torch_lstmcell():
    rng = np.random.default_rng(1)
    n_in, n_h, n = 7, 5, 4
    w_ih, w_hh = rng.normal(size=(4 * n_h, n_in)), rng.normal(size=(4 * n_h, n_h))
    b_ih, b_hh = rng.normal(size=4 * n_h), rng.normal(size=4 * n_h)
    u, h, c = rng.normal(size=(n, n_in)), rng.normal(size=(n, n_h)), rng.normal(size=(n, n_h))
    cell = torch.nn.LSTMCell(n_in, n_h).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(w_ih)); cell.weight_hh.copy_(torch.from_numpy(w_hh))
        cell.bias_ih.copy_(torch.from_numpy(b_ih)); cell.bias_hh.copy_(torch.from_numpy(b_hh))
        h_ref, c_ref = cell(torch.from_numpy(u), (torch.from_numpy(h), torch.from_numpy(c)))
    h_o, c_o = lstm_cell(w_ih, w_hh, b_ih, b_hh, u, h, c)
    np.testing.assert_allclose(h_o, h_ref.numpy(), atol=1e-14)
    np.testing.assert_allclose(c_o, c_ref.numpy(), atol=1e-14)


@pytest.mark.parametrize("cfg", [SMALL, SMALL_BI, synth.ModelConfig(3, 5, 6, 9, 9, True, True)])
def test_encoder_matches_torch_packed_lstm(cfg):
    m = toy_model(cfg, seed=5, scale=0.5)
    D = 2 if cfg.bidir else 1
    lstm = torch.nn.LSTM(cfg.emb, cfg.h_dir, num_layers=cfg.layers, bidirectional=cfg.bidir,
                         batch_first=True).double()
    with torch.no_grad():
        for l in range(cfg.layers):
            for d, sfx in zip(["fwd", "bwd"][:D], ["", "_reverse"]):
                p = f"enc.l{l}.{d}."
                getattr(lstm, f"weight_ih_l{l}{sfx}").copy_(torch.from_numpy(m.t[p + "w_ih"]))
                getattr(lstm, f"weight_hh_l{l}{sfx}").copy_(torch.from_numpy(m.t[p + "w_hh"]))
                getattr(lstm, f"bias_ih_l{l}{sfx}").copy_(torch.from_numpy(m.t[p + "b_ih"]))
                getattr(lstm, f"bias_hh_l{l}{sfx}").copy_(torch.from_numpy(m.t[p + "b_hh"]))
    lens = [7, 3, 1, 5]
    rng = np.random.default_rng(2)
    ids = np.zeros((4, 7), np.int64)
    for b, L in enumerate(lens):
        ids[b, :L] = rng.integers(4, cfg.v_src, L)
        ids[b, L:] = rng.integers(0, cfg.v_src, 7 - L)        # garbage at pads must not matter
    x = torch.from_numpy(m.emb_src[ids])
    packed = torch.nn.utils.rnn.pack_padded_sequence(x, torch.tensor(lens), batch_first=True,
                                                     enforce_sorted=False)
    with torch.no_grad():
        out, (h_n, c_n) = lstm(packed)
    out, _ = torch.nn.utils.rnn.pad_packed_sequence(out, batch_first=True)
    h_n = h_n.view(cfg.layers, D, 4, cfg.h_dir)
    c_n = c_n.view(cfg.layers, D, 4, cfg.h_dir)
    for b, L in enumerate(lens):
        mem, finals = m.encode(list(ids[b, :L]))
        np.testing.assert_allclose(mem, out[b, :L].numpy(), atol=1e-13)
        for l in range(cfg.layers):
            np.testing.assert_allclose(finals[l][0], h_n[l, :, b].reshape(-1).numpy(), atol=1e-13)
            np.testing.assert_allclose(finals[l][1], c_n[l, :, b].reshape(-1).numpy(), atol=1e-13)


def test_lstm_zero_weights_closed_form():
    n = 6
    z4, z = np.zeros((4 * n, n)), np.zeros(4 * n)
    rng = np.random.default_rng(3)
    h, c0 = np.zeros(n), rng.normal(size=n)
    c = c0.copy()
    for t in range(1, 9):
        h, c = lstm_cell(z4, z4, z, z, rng.normal(size=n), h, c)   # i=f=o=1/2, g=0
        np.testing.assert_allclose(c, 0.5 ** t * c0, rtol=1e-15)
        np.testing.assert_allclose(h, 0.5 * np.tanh(0.5 ** t * c0), rtol=1e-15)
    # all zero and zero start -> stays zero
    h, c = lstm_cell(z4, z4, z, z, rng.normal(size=n), np.zeros(n), np.zeros(n))
    assert not h.any() and not c.any()


def test_encoder_bias_only_closed_form_catches_gate_order_and_packing():
    """W = 0, b != 0: c_t = i g (1 - f^t)/(1 - f), h_t = o tanh(c_t) with
    i = s(b_i), f = s(b_f), g = tanh(b_g), o = s(b_o) (distinct per gate)."""
    cfg = synth.ModelConfig(1, 4, 5, 20, 20, False, True)
    base = {k: np.zeros_like(v, dtype=np.float64) for k, v in synth.random_model_tensors(cfg, 0).items()}
    H = 5
    b = np.concatenate([np.full(H, 0.3), np.full(H, -0.7), np.full(H, 1.1), np.full(H, 0.2)])
    base["enc.l0.fwd.b_ih"] = b / 2
    base["enc.l0.fwd.b_hh"] = b / 2
    base["enc.emb"] = np.random.default_rng(0).normal(size=(20, 4))
    m = OracleModel(base)
    s = lambda x: 1 / (1 + math.exp(-x))
    i, f, g, o = s(0.3), s(-0.7), math.tanh(1.1), s(0.2)
    for S in (8, 5, 1):
        mem, finals = m.encode(list(range(4, 4 + S)))
        ct = i * g * (1 - f ** S) / (1 - f)
        np.testing.assert_allclose(finals[0][1], ct, rtol=1e-14)
        np.testing.assert_allclose(finals[0][0], o * math.tanh(ct), rtol=1e-14)
        for t in range(S):
            ctt = i * g * (1 - f ** (t + 1)) / (1 - f)
            np.testing.assert_allclose(mem[t], o * math.tanh(ctt), rtol=1e-14)


# ------------------------------------------------------------------ attention
def test_attention_invariants():
    m = toy_model(SMALL, seed=7, scale=0.5)
    rng = np.random.default_rng(4)
    mem = rng.normal(size=(9, SMALL.hidden))
    h = rng.normal(size=(3, SMALL.hidden))
    for L in (9, 4, 1):
        a, ctx = m.attention(h, mem, L)
        np.testing.assert_allclose(a.sum(axis=1), 1.0, atol=1e-12)
        assert (a[:, L:] == 0).all() and (a >= 0).all()
        # loop form (S283) as an independent restatement
        q = h @ m.t["attn.w_in"].T
        for n in range(3):
            e = [sum(q[n, j] * mem[s, j] for j in range(SMALL.hidden)) for s in range(L)]
            mx = max(e)
            w = [math.exp(v - mx) for v in e]
            w = [v / sum(w) for v in w]
            c = [sum(w[s] * mem[s, j] for s in range(L)) for j in range(SMALL.hidden)]
            np.testing.assert_allclose(a[n, :L], w, atol=1e-12)
            np.testing.assert_allclose(ctx[n], c, atol=1e-12)
    # S = 1 -> [1.0] and c = m_0 (S273)
    a, ctx = m.attention(h, mem, 1)
    assert a[0, 0] == golden("attn_single")[0]
    np.testing.assert_array_equal(ctx[0], mem[0])
    # softmax([1,1]) = [.5,.5] (S45): two identical memory rows
    a, _ = m.attention(h, np.stack([mem[0], mem[0]]), 2)
    np.testing.assert_allclose(a[0], golden("softmax_11"), atol=1e-15)
    # permuting memory rows permutes weights and leaves the context unchanged
    perm = rng.permutation(9)
    a1, c1 = m.attention(h, mem, 9)
    a2, c2 = m.attention(h, mem[perm], 9)
    np.testing.assert_allclose(a2, a1[:, perm], atol=1e-14)
    np.testing.assert_allclose(c2, c1, atol=1e-13)


def test_attention_special_cases():
    rng = np.random.default_rng(5)
    mem = rng.normal(size=(6, SMALL.hidden))
    h = rng.normal(size=(2, SMALL.hidden))
    m0 = toy_model(SMALL, overrides={"attn.w_in": np.zeros((8, 8))})
    a, ctx = m0.attention(h, mem, 5)
    np.testing.assert_allclose(a[:, :5], 1 / 5, atol=1e-15)
    np.testing.assert_allclose(ctx, np.tile(mem[:5].mean(axis=0), (2, 1)), atol=1e-14)
    mi = toy_model(SMALL, overrides={"attn.w_in": np.eye(8)})
    md = toy_model(SMALL_BI)      # dot
    ai, ci = mi.attention(h, mem, 6)
    ad, cd = md.attention(h, mem, 6)
    np.testing.assert_allclose(ai, ad, atol=1e-15)
    np.testing.assert_allclose(ci, cd, atol=1e-15)
    # zero query, dot -> uniform (S272)
    a0, _ = md.attention(np.zeros((1, 8)), mem, 6)
    np.testing.assert_allclose(a0[0], 1 / 6, atol=1e-15)


# ------------------------------------------------------------------ decode step / generator
def _step(m, src, y=(2,), ht=None):
    mem, finals = m.encode(src)
    y0, ht0, st = m.init_decoder(finals, len(y))
    return m.decode_step(np.array(y), ht0 if ht is None else ht, st, mem)


def test_generator_zero_weights_uniform_exact():
    cfg = synth.ModelConfig(1, 4, 6, 100, 100, False, True)
    m = toy_model(cfg, overrides={"gen.w": np.zeros((100, 6)), "gen.b": np.zeros(100)})
    logp = _step(m, [5, 6, 7])[0]
    assert (logp == golden("zero_generator")[0]).all()
    assert (logp == -math.log(100)).all()


def test_generator_wout_zero_equals_scipy_log_softmax_of_bias():
    cfg = synth.ModelConfig(2, 4, 6, 30, 40, False, True)
    m = toy_model(cfg, seed=1, scale=1.0, overrides={"attn.w_out": np.zeros((6, 12))})
    ref = scipy.special.log_softmax(m.t["gen.b"])
    for src in ([5, 6, 7], [9]):
        logp = _step(m, src, y=(2, 7, 3))[0]
        np.testing.assert_allclose(logp, np.tile(ref, (3, 1)), atol=1e-14)


def test_log_probs_normalised():
    m = toy_model(SMALL, seed=2, scale=2.0)
    logp = _step(m, [4, 5, 6, 7], y=(2, 5))[0]
    np.testing.assert_allclose(scipy.special.logsumexp(logp, axis=1), 0.0, atol=1e-12)


def test_htilde_context_first_and_input_feed_columns():
    cfg = synth.ModelConfig(1, 4, 6, 20, 20, False, True)
    H = 6
    rng = np.random.default_rng(9)
    # W_out = [0 | I]: h~ = tanh(h_t) -> output independent of the memory bank
    m = toy_model(cfg, seed=3, scale=1.0, overrides={"attn.w_out": np.hstack([np.zeros((H, H)), np.eye(H)])})
    mem_a, fin = m.encode([4, 5, 6])
    y, ht, st = m.init_decoder(fin, 1)
    la = m.decode_step(y, ht, st, mem_a)[0]
    lb = m.decode_step(y, ht, st, rng.normal(size=mem_a.shape))[0]
    np.testing.assert_allclose(la, lb, atol=1e-14)
    # W_out = [I | 0] with S=1: h~ = tanh(m_0) -> logp = log_softmax(W_gen tanh(m_0) + b)
    m2 = toy_model(cfg, seed=3, scale=1.0, overrides={"attn.w_out": np.hstack([np.eye(H), np.zeros((H, H))])})
    mem, fin = m2.encode([7])
    y, ht, st = m2.init_decoder(fin, 1)
    lp = m2.decode_step(y, ht, st, mem)[0]
    ref = scipy.special.log_softmax(m2.t["gen.w"] @ np.tanh(mem[0]) + m2.t["gen.b"])
    np.testing.assert_allclose(lp[0], ref, atol=1e-13)
    # input-feed columns (E..E+H) zero -> independent of h~_prev (S291 ablation)
    w = m.t["dec.l0.w_ih"].copy(); w[:, 4:] = 0
    m3 = toy_model(cfg, seed=3, scale=1.0, overrides={"dec.l0.w_ih": w})
    mem, fin = m3.encode([4, 5])
    y, ht, st = m3.init_decoder(fin, 1)
    l1 = m3.decode_step(y, ht, st, mem)[0]
    l2 = m3.decode_step(y, rng.normal(size=ht.shape), st, mem)[0]
    np.testing.assert_allclose(l1, l2, atol=1e-14)
    # embedding columns zero -> independent of y_prev
    w = m.t["dec.l0.w_ih"].copy(); w[:, :4] = 0
    m4 = toy_model(cfg, seed=3, scale=1.0, overrides={"dec.l0.w_ih": w})
    mem, fin = m4.encode([4, 5])
    y, ht, st = m4.init_decoder(fin, 1)
    np.testing.assert_allclose(m4.decode_step(np.array([2]), ht, st, mem)[0],
                               m4.decode_step(np.array([9]), ht, st, mem)[0], atol=1e-14)


def test_decode_step_rows_independent():
    m = toy_model(SMALL_BI, seed=4, scale=0.8)
    mem, fin = m.encode([4, 8, 9, 10])
    y, ht, st = m.init_decoder(fin, 3)
    rng = np.random.default_rng(1)
    ht = rng.normal(size=ht.shape)
    st = [(h + rng.normal(size=h.shape), c + rng.normal(size=c.shape)) for h, c in st]
    yy = np.array([2, 7, 10])
    full = m.decode_step(yy, ht, st, mem)[0]
    for r in range(3):
        one = m.decode_step(yy[r:r + 1], ht[r:r + 1], [(h[r:r + 1], c[r:r + 1]) for h, c in st], mem)[0]
        np.testing.assert_allclose(one[0], full[r], atol=1e-14)


def test_decoder_step_matches_torch_modules():
    """Independent torch fp64 restatement of one decode step with nn.LSTMCell,
    F.log_softmax and explicit masked softmax (library cross-check)."""
    cfg = synth.ModelConfig(2, 5, 6, 15, 17, False, True)
    m = toy_model(cfg, seed=11, scale=0.7)
    mem, fin = m.encode([4, 5, 6, 7])
    y, ht, st = m.init_decoder(fin, 2)
    y = np.array([2, 9])
    ht = np.random.default_rng(0).normal(size=(2, 6))
    logp, a, ht_new, _ = m.decode_step(y, ht, st, mem)
    T = lambda x: torch.from_numpy(np.asarray(x))
    cells = []
    for l in range(2):
        c = torch.nn.LSTMCell(5 + 6 if l == 0 else 6, 6).double()
        with torch.no_grad():
            c.weight_ih.copy_(T(m.t[f"dec.l{l}.w_ih"])); c.weight_hh.copy_(T(m.t[f"dec.l{l}.w_hh"]))
            c.bias_ih.copy_(T(m.t[f"dec.l{l}.b_ih"])); c.bias_hh.copy_(T(m.t[f"dec.l{l}.b_hh"]))
        cells.append(c)
    with torch.no_grad():
        x = torch.cat([T(m.t["dec.emb"][y]), T(ht)], 1)
        for l in range(2):
            h, c = cells[l](x, (T(st[l][0]), T(st[l][1])))
            x = h
        q = torch.nn.functional.linear(x, T(m.t["attn.w_in"]))
        att = torch.softmax(q @ T(mem).T, dim=1)
        ctx = att @ T(mem)
        hh = torch.tanh(torch.nn.functional.linear(torch.cat([ctx, x], 1), T(m.t["attn.w_out"])))
        lp = torch.log_softmax(torch.nn.functional.linear(hh, T(m.t["gen.w"]), T(m.t["gen.b"])), 1)
    np.testing.assert_allclose(logp, lp.numpy(), atol=1e-13)
    np.testing.assert_allclose(ht_new, hh.numpy(), atol=1e-14)
    np.testing.assert_allclose(a, att.numpy(), atol=1e-14)
