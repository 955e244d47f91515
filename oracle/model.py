"""fp64 attention-based LSTM encoder-decoder (oracle).  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2 (P105-139) and the readings in DESIGN.md §3 (SURVEY.md
§8(c) AMB-1..AMB-11).  Plain numpy, float64 throughout; a matrix-vector or
matrix-matrix product (`@`) is the only library primitive used.

Notation: E embedding width, H decoder width (= memory width), Hd per-direction
encoder width, L layers, V target vocabulary.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

PAD, UNK, BOS, EOS = 0, 1, 2, 3


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Logistic function 1/(1+e^-x), written in the overflow-safe two-branch form."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def lstm_cell(w_ih, w_hh, b_ih, b_hh, u, h, c):
    """One LSTM step (P129-131 "gated RNN such as an LSTM"; O2; AMB-1).

    z = W_ih u + b_ih + W_hh h + b_hh, row blocks (i, f, g, o);
    i, f, o = sigmoid; g = tanh; c' = f*c + i*g; h' = o*tanh(c').
    u, h, c may be vectors or [n x .] row stacks."""
    z = u @ w_ih.T + b_ih + h @ w_hh.T + b_hh
    n = w_hh.shape[1]
    i = sigmoid(z[..., 0 * n:1 * n])
    f = sigmoid(z[..., 1 * n:2 * n])
    g = np.tanh(z[..., 2 * n:3 * n])
    o = sigmoid(z[..., 3 * n:4 * n])
    c_new = f * c + i * g
    h_new = o * np.tanh(c_new)
    return h_new, c_new


def log_softmax(z: np.ndarray) -> np.ndarray:
    """log p = z - (max z + log sum exp(z - max z)) over the last axis
    (P118-119 "A softmax layer"; SPEC S76 max-subtraction; O6)."""
    m = np.max(z, axis=-1, keepdims=True)
    return z - (m + np.log(np.sum(np.exp(z - m), axis=-1, keepdims=True)))


class OracleModel:
    """Weights (fp64 dict from `mnmt.load_model_tensors`) plus the forward pieces."""

    def __init__(self, t: Dict[str, np.ndarray]):
        self.t = t
        self.emb_src = t["enc.emb"]
        self.emb_tgt = t["dec.emb"]
        self.E = self.emb_src.shape[1]
        self.bidir = "enc.l0.bwd.w_ih" in t
        self.L = 0
        while f"dec.l{self.L}.w_ih" in t:
            self.L += 1
        self.H = t["dec.l0.w_hh"].shape[1]
        self.Hd = t["enc.l0.fwd.w_hh"].shape[1]
        self.general = "attn.w_in" in t
        self.V = t["gen.w"].shape[0]
        self.copy = "copy.w" in t            # copy / pointer generator (SPEC S293-301)
        self.dirs = ["fwd", "bwd"] if self.bidir else ["fwd"]
        assert self.Hd * len(self.dirs) == self.H, "AMB-5: [fwd;bwd] must equal the decoder width"

    # ---------------------------------------------------------------- encoder
    def enc_params(self, l: int, d: str):
        p = f"enc.l{l}.{d}."
        t = self.t
        return t[p + "w_ih"], t[p + "w_hh"], t[p + "b_ih"], t[p + "b_hh"]

    def dec_params(self, l: int):
        p = f"dec.l{l}."
        t = self.t
        return t[p + "w_ih"], t[p + "w_hh"], t[p + "b_ih"], t[p + "b_hh"]

    def encode(self, src: List[int]):
        """O2/O3 for ONE sentence of S_b tokens (P112-115 "maps each source word
        to a word vector, and processes these to a sequence of hidden vectors";
        P131-133 stacked layers; AMB-3 packed semantics, AMB-6 stacked biLSTM).

        Returns (memory [S_b x H], init [(h, c) per decoder layer])."""
        S = len(src)
        if S < 1:
            raise ValueError("empty source (S431)")
        inp = self.emb_src[np.asarray(src, dtype=np.int64)]          # [S x E]
        finals = []
        for l in range(self.L):
            outs, hs, cs = [], [], []
            for d in self.dirs:
                w_ih, w_hh, b_ih, b_hh = self.enc_params(l, d)
                h = np.zeros(self.Hd)
                c = np.zeros(self.Hd)
                out = np.zeros((S, self.Hd))
                order = range(S) if d == "fwd" else range(S - 1, -1, -1)
                for t in order:
                    h, c = lstm_cell(w_ih, w_hh, b_ih, b_hh, inp[t], h, c)
                    out[t] = h
                outs.append(out)
                hs.append(h)   # fwd: state after t = S_b-1; bwd: after t = 0
                cs.append(c)
            inp = np.concatenate(outs, axis=1)                       # [S x D*Hd]
            finals.append((np.concatenate(hs), np.concatenate(cs)))  # AMB-5
        return inp, finals

    # -------------------------------------------------------------- attention
    def attention(self, h_t: np.ndarray, memory: np.ndarray, length: int | None = None):
        """Luong global attention, O5 (P119-122 "attention pooling layer that
        weights each source word"; P299-301 general / dot; AMB-8).

        h_t [n x H]; memory [S_pad x H]; positions s >= length are pads.
        Returns (a [n x S_pad] with a == 0 exactly at pads, context [n x H])."""
        S_pad = memory.shape[0]
        length = S_pad if length is None else length
        q = h_t @ self.t["attn.w_in"].T if self.general else h_t     # q = W_in h_t
        e = q @ memory[:length].T                                     # e_s = q . m_s
        m = np.max(e, axis=-1, keepdims=True)
        ex = np.exp(e - m)
        a_real = ex / np.sum(ex, axis=-1, keepdims=True)
        a = np.zeros((h_t.shape[0], S_pad))
        a[:, :length] = a_real
        ctx = a_real @ memory[:length]                                # c = sum a_s m_s
        return a, ctx

    # ------------------------------------------------------------ decode step
    def decode_step(self, y_prev: np.ndarray, htilde_prev: np.ndarray,
                    states: List[Tuple[np.ndarray, np.ndarray]], memory: np.ndarray):
        """O4-O6 for n hypotheses of ONE sentence.

        Input feeding (P133-136): u = [E_tgt[y_prev] ; h~_prev] (AMB-7).
        Stacked decoder LSTM (P115-118, P131-133).  Attention (O5).
        h~ = tanh(W_out [c ; h_t]) (P69 "combined with the current hidden
        state"; AMB-9, no bias).  Generator z = W_gen h~ + b, log-softmax over
        all V ids (P118-119; AMB-10/11).

        Returns (logp [n x V], attn [n x S], h~ [n x H], new states)."""
        u = np.concatenate([self.emb_tgt[np.asarray(y_prev, dtype=np.int64)], htilde_prev], axis=1)
        new_states = []
        x = u
        for l in range(self.L):
            h, c = states[l]
            h, c = lstm_cell(*self.dec_params(l), x, h, c)
            new_states.append((h, c))
            x = h
        h_top = x
        a, ctx = self.attention(h_top, memory)
        htilde = np.tanh(np.concatenate([ctx, h_top], axis=1) @ self.t["attn.w_out"].T)
        z = htilde @ self.t["gen.w"].T + self.t["gen.b"]
        return log_softmax(z), a, htilde, new_states

    # ------------------------------------------------------------- copy model
    def copy_gate(self, htilde: np.ndarray) -> np.ndarray:
        """g = sigmoid(w_copy . h~ + b_copy) per hypothesis: the generator's share of the
        extended distribution (SPEC S293-297 "copy_gate"; reading DESIGN.md §3 R31)."""
        return sigmoid(htilde @ self.t["copy.w"][0] + self.t["copy.b"][0])

    @staticmethod
    def extended_log_probs(logp: np.ndarray, a: np.ndarray, g: np.ndarray, src_ext: List[int],
                           v_ext: int) -> np.ndarray:
        """S296: p(w) = g p_vocab(w) + (1 - g) sum_{s: src_s = w} a_s over the extended
        vocabulary (target vocabulary, then this sentence's source-only ids).
        logp [n x V] generator log-probs, a [n x S] attention, g [n], src_ext [S] ids."""
        n, V = logp.shape
        p = np.zeros((n, v_ext))
        p[:, :V] = g[:, None] * np.exp(logp)
        for s, w in enumerate(src_ext):                 # scatter-add of the copy attention
            p[:, w] += (1.0 - g) * a[:, s]
        with np.errstate(divide="ignore"):
            return np.log(p)

    def init_decoder(self, finals, n: int):
        """O3: decoder layer l starts from the encoder layer-l final state,
        replicated to n rows; h~_0 = 0; y_0 = BOS."""
        states = [(np.tile(h, (n, 1)), np.tile(c, (n, 1))) for (h, c) in finals]
        return np.full(n, BOS, dtype=np.int64), np.zeros((n, self.H)), states
