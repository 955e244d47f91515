"""Beam search, greedy, brute force and teacher-forced scoring (oracle).

TEST INFRASTRUCTURE ONLY.  PAPER.md P136-139 (§2(d) "Test-time decoding is
done through beam search where multiple hypothesis target predictions are
considered at each time step"), P315-316 (length normalisation, citing GNMT),
SPEC.md S427-444; the step-by-step rule is SURVEY.md §8(c) O7-O11 with the
readings AMB-12..AMB-19.
"""
from __future__ import annotations

import itertools
from typing import Dict, List, Optional

import numpy as np

from .model import BOS, EOS, UNK, OracleModel

TRACE_MARGIN = 16


def length_penalty(n: int, alpha: float) -> float:
    """GNMT lp(n) = ((5 + n) / 6)^alpha (S439; P315-316; AMB-17: n counts EOS)."""
    return ((5.0 + n) / 6.0) ** alpha


def coverage_penalty(cum_attn: np.ndarray, beta: float) -> float:
    """GNMT cp = beta * sum_s log(min(sum_t a_{t,s}, 1.0)) over the real source
    positions (S439 final_score; P315-316 "attention coverage normalization", formula of
    the cited GNMT reference, SPEC S489).  cum_attn = sum over the hypothesis's steps
    (every emitted token, EOS included) of its attention weights.  beta = 0 -> 0."""
    if beta == 0.0:
        return 0.0
    return float(beta * np.sum(np.log(np.minimum(cum_attn, 1.0))))


def final_score(raw: float, n: int, cum_attn: np.ndarray, alpha: float, beta: float) -> float:
    """S436-439 final_score(hyp, alpha, beta) = raw / lp(|Y|) + cp."""
    return raw / length_penalty(n, alpha) + coverage_penalty(cum_attn, beta)


def replace_unknowns(tokens: List[int], attn_argmax: List[int]) -> List[int]:
    """S445-448 in id space: for every <unk> (id 1) emitted at step t, the source
    POSITION argmax_s a_{t,s} (ties -> smallest s) whose word replaces it; -1 for every
    other token (no phrase table: the caller copies the source word at that position)."""
    return [int(j) if w == UNK else -1 for w, j in zip(tokens, attn_argmax)]


def _select(cum: np.ndarray, live: np.ndarray, logp: np.ndarray, K: int, M: int):
    """O8 candidate ranking: every (k, w) with k live, score s = cum_k + logp[k, w],
    ordered by (s desc, k asc, w asc) (AMB-13).  Returns the first K + M entries
    as (s, k, w) tuples; selection is the first min(K, #candidates).

    Exact top-(K+M): keep every candidate whose score is >= the (K+M)-th largest
    score (ties included), then sort that subset with the full key."""
    ks = np.nonzero(live)[0]
    scores = cum[ks][:, None] + logp[ks]                   # [n_live x V]
    flat = scores.ravel()
    need = min(K + M, flat.size)
    thr = np.partition(flat, flat.size - need)[flat.size - need]
    idx = np.nonzero(flat >= thr)[0]
    kk = ks[idx // logp.shape[1]]
    ww = idx % logp.shape[1]
    ss = flat[idx]
    order = np.lexsort((ww, kk, -ss))                      # last key is primary
    return [(float(ss[i]), int(kk[i]), int(ww[i])) for i in order[:need]]


def _step_log_probs(model: OracleModel, y, htilde, states, memory, src_ext):
    """One decoder step for the hypotheses of one sentence: (log p over the vocabulary -
    extended by the sentence's source-only ids for a copy model, S293-297 -, attention,
    h~, states).  A copy model reads an emitted extended id >= V back as <unk> (R32)."""
    y_in = np.where(np.asarray(y) < model.V, y, UNK)
    logp, a, ht, st = model.decode_step(y_in, htilde, states, memory)
    if model.copy:
        v_ext = max(model.V, max(src_ext) + 1)
        logp = model.extended_log_probs(logp, a, model.copy_gate(ht), src_ext, v_ext)
    return logp, a, ht, st


def beam_search(model: OracleModel, src: List[int], K: int, max_len: int, alpha: float = 0.0,
                stop: str = "rank0", trace: bool = False, beta: float = 0.0, n_best: int = 1,
                src_ext: Optional[List[int]] = None) -> Dict:
    """O7-O11 for one sentence.

    beta > 0: banked entries are scored by final_score (raw / lp + cp, S436-439); the
    ranking inside a step stays by raw score (AMB-13).  n_best: the returned "nbest"
    list holds the n best bank entries (S422-423, 1 <= n_best <= K) in final order.
    Every hypothesis carries its cumulative attention and the per-token attention
    argmax (for coverage and unknown-word replacement, S445-448).

    stop = "rank0": stop after step t if the rank-0 selection is EOS, or no slot
             is live, or t == max_len (O10, AMB-15) - the product rule.
    stop = "bound": S480's rule - stop when the best banked normalised score is
             >= max over live slots of cum / lp(max_len) (a valid upper bound
             since log p <= 0), or nothing is live, or t == max_len.
    stop = "none": only the no-live and max_len stops.
    """
    if K < 1 or max_len < 1:
        raise ValueError("beam and max_len must be >= 1")
    if not 1 <= n_best <= K:
        raise ValueError("1 <= n_best <= beam (S423)")
    if model.copy and (src_ext is None or len(src_ext) != len(src)):
        raise ValueError("a copy model needs src_ext: one extended id per source position (S293)")
    memory, finals = model.encode(src)
    y0, ht0, st0 = model.init_decoder(finals, 1)
    H = model.H
    # slot arrays (O7): only slot 0 is live at t = 1 (AMB-12)
    live = np.zeros(K, dtype=bool); live[0] = True
    cum = np.full(K, -np.inf); cum[0] = 0.0
    y = np.full(K, BOS, dtype=np.int64)
    htilde = np.zeros((K, H))
    states = [(np.zeros((K, H)), np.zeros((K, H))) for _ in range(model.L)]
    for l in range(model.L):
        states[l][0][0] = st0[l][0][0]
        states[l][1][0] = st0[l][1][0]
    hyps: List[List[int]] = [[] for _ in range(K)]
    lps: List[List[float]] = [[] for _ in range(K)]
    S = len(src)
    catt = np.zeros((K, S))                                    # cumulative attention per slot
    amax: List[List[int]] = [[] for _ in range(K)]             # per-token attention argmax
    bank = []      # (norm, t, r, raw, hyp, lps, amax, cp)
    steps = []
    for t in range(1, max_len + 1):
        ks = np.nonzero(live)[0]
        logp_l, att_l, ht_l, st_l = _step_log_probs(
            model, y[ks], htilde[ks], [(h[ks], c[ks]) for (h, c) in states], memory, src_ext)
        logp = np.full((K, logp_l.shape[1]), -np.inf)
        logp[ks] = logp_l
        cand = _select(cum, live, logp, K, TRACE_MARGIN)
        n_sel = min(K, int(live.sum()) * model.V)
        sel = cand[:n_sel]
        # O8: selected entry r becomes slot r at t+1, state of its parent k
        n_live = np.zeros(K, dtype=bool)
        n_cum = np.full(K, -np.inf)
        n_y = np.full(K, BOS, dtype=np.int64)
        n_ht = np.zeros((K, H))
        n_states = [(np.zeros((K, H)), np.zeros((K, H))) for _ in range(model.L)]
        n_hyps: List[List[int]] = [[] for _ in range(K)]
        n_lps: List[List[float]] = [[] for _ in range(K)]
        n_catt = np.zeros((K, S))
        n_amax: List[List[int]] = [[] for _ in range(K)]
        pos = {int(k): i for i, k in enumerate(ks)}
        for r, (s, k, w) in enumerate(sel):
            i = pos[k]
            n_hyps[r] = hyps[k] + [w]
            n_lps[r] = lps[k] + [float(logp[k, w])]
            n_catt[r] = catt[k] + att_l[i]                     # a_t of the parent's step-t state
            n_amax[r] = amax[k] + [int(np.argmax(att_l[i]))]   # first maximum: ties -> smallest s
            if w == EOS or t == max_len:                       # O9 banking
                n = t
                cp = coverage_penalty(n_catt[r], beta)
                bank.append((final_score(s, n, n_catt[r], alpha, beta), t, r, s, n_hyps[r], n_lps[r],
                             n_amax[r], cp))
            else:
                n_live[r] = True
                n_cum[r] = s
                n_y[r] = w
                n_ht[r] = ht_l[i]
                for l in range(model.L):
                    n_states[l][0][r] = st_l[l][0][i]
                    n_states[l][1][r] = st_l[l][1][i]
        if trace:
            steps.append({"t": t, "cand": cand, "sel": [(k, w, s) for (s, k, w) in sel],
                          "cum": cum.copy(), "live": live.copy()})
        live, cum, y, htilde, states, hyps, lps = n_live, n_cum, n_y, n_ht, n_states, n_hyps, n_lps
        catt, amax = n_catt, n_amax
        # O10 stop
        if not live.any() or t == max_len:
            break
        if stop == "rank0" and sel[0][2] == EOS:
            break
        if stop == "bound" and bank:
            best_norm = max(b[0] for b in bank)
            bound = max(cum[k] / length_penalty(max_len, alpha) for k in np.nonzero(live)[0])
            if best_norm >= bound:
                break
    if not bank:
        raise RuntimeError("beam exhausted with empty bank (S431)")
    # O11: largest norm; ties -> smaller t, then smaller r (AMB-19)
    ranked = sorted(bank, key=lambda b: (-b[0], b[1], b[2]))
    best = ranked[0]
    out = {"tokens": list(best[4]), "norm": best[0], "raw": best[3], "t": best[1], "r": best[2],
           "token_logp": list(best[5]), "attn_argmax": list(best[6]), "cp": best[7], "bank": bank,
           "nbest": [{"tokens": list(e[4]), "norm": e[0], "raw": e[3], "t": e[1], "r": e[2],
                      "token_logp": list(e[5]), "attn_argmax": list(e[6]), "cp": e[7]}
                     for e in ranked[:n_best]]}
    if trace:
        out["steps"] = steps
    return out


def greedy(model: OracleModel, src: List[int], max_len: int, src_ext: Optional[List[int]] = None) -> Dict:
    """O12: argmax with the lowest id on ties; stop at EOS or max_len."""
    memory, finals = model.encode(src)
    y, ht, st = model.init_decoder(finals, 1)
    toks, lps = [], []
    for t in range(1, max_len + 1):
        logp, _, ht, st = _step_log_probs(model, y, ht, st, memory, src_ext)
        w = int(np.argmax(logp[0]))          # np.argmax returns the first maximum
        toks.append(w); lps.append(float(logp[0, w]))
        y = np.array([w])
        if w == EOS:
            break
    return {"tokens": toks, "raw": float(np.sum(lps)), "token_logp": lps}


def score_sequence(model: OracleModel, src: List[int], Y: List[int], with_attn: bool = False,
                   src_ext: Optional[List[int]] = None):
    """Teacher-forced log p(y_t | y_<t, x) of every token of Y (P105-108); with_attn:
    also the attention rows a_t [|Y| x S] of those steps."""
    memory, finals = model.encode(src)
    y, ht, st = model.init_decoder(finals, 1)
    out, att = [], []
    for w in Y:
        logp, a, ht, st = _step_log_probs(model, y, ht, st, memory, src_ext)
        out.append(float(logp[0, w]))
        att.append(a[0])
        y = np.array([w])
    return (out, np.array(att)) if with_attn else out


def brute_force(model: OracleModel, src: List[int], max_len: int, alpha: float = 0.0,
                beta: float = 0.0, src_ext: Optional[List[int]] = None) -> List[Dict]:
    """O12: enumerate Y = {sequences ending at their first EOS, length <= max_len}
    U {EOS-free sequences of length exactly max_len}; score each by teacher
    forcing (final_score: raw / lp + cp).  Returns all of them sorted by (norm desc,
    then token tuple)."""
    V = max(model.V, max(src_ext) + 1) if model.copy else model.V
    out = []
    for n in range(1, max_len + 1):
        for prefix in itertools.product([w for w in range(V) if w != EOS], repeat=n - 1):
            tails = [EOS] if n < max_len else list(range(V))
            for last in tails:
                Y = list(prefix) + [last]
                lp, att = score_sequence(model, src, Y, with_attn=True, src_ext=src_ext)
                raw = float(np.sum(lp))
                out.append({"tokens": Y, "raw": raw, "norm": final_score(raw, n, att.sum(0), alpha, beta),
                            "token_logp": lp})
    out.sort(key=lambda d: (-d["norm"], d["tokens"]))
    return out


def translate_batch(model: OracleModel, srcs: List[List[int]], K: int, max_len: int,
                    alpha: float = 0.0, trace: bool = False) -> List[Dict]:
    """S463-471: every sentence decoded independently (batching is a pure
    optimisation, S466); an empty batch gives an empty result (S471)."""
    return [beam_search(model, s, K, max_len, alpha, trace=trace) for s in srcs]


def unpad(ids: np.ndarray, lens: np.ndarray) -> List[List[int]]:
    return [list(map(int, ids[b, : lens[b]])) for b in range(len(lens))]


def model_from_file(path: str, precision: str) -> OracleModel:
    from .mnmt import load_model_tensors
    return OracleModel(load_model_tensors(path, precision))


__all__ = ["beam_search", "greedy", "score_sequence", "brute_force", "translate_batch",
           "length_penalty", "coverage_penalty", "final_score", "replace_unknowns", "unpad",
           "model_from_file", "Optional"]
