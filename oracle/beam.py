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

from .model import BOS, EOS, OracleModel

TRACE_MARGIN = 16


def length_penalty(n: int, alpha: float) -> float:
    """GNMT lp(n) = ((5 + n) / 6)^alpha (S439; P315-316; AMB-17: n counts EOS)."""
    return ((5.0 + n) / 6.0) ** alpha


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


def beam_search(model: OracleModel, src: List[int], K: int, max_len: int, alpha: float = 0.0,
                stop: str = "rank0", trace: bool = False) -> Dict:
    """O7-O11 for one sentence.

    stop = "rank0": stop after step t if the rank-0 selection is EOS, or no slot
             is live, or t == max_len (O10, AMB-15) - the product rule.
    stop = "bound": S480's rule - stop when the best banked normalised score is
             >= max over live slots of cum / lp(max_len) (a valid upper bound
             since log p <= 0), or nothing is live, or t == max_len.
    stop = "none": only the no-live and max_len stops.
    """
    if K < 1 or max_len < 1:
        raise ValueError("beam and max_len must be >= 1")
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
    bank = []      # (norm, t, r, raw, hyp, lps)
    steps = []
    for t in range(1, max_len + 1):
        ks = np.nonzero(live)[0]
        logp_l, _, ht_l, st_l = model.decode_step(
            y[ks], htilde[ks], [(h[ks], c[ks]) for (h, c) in states], memory)
        logp = np.full((K, model.V), -np.inf)
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
        pos = {int(k): i for i, k in enumerate(ks)}
        for r, (s, k, w) in enumerate(sel):
            i = pos[k]
            n_hyps[r] = hyps[k] + [w]
            n_lps[r] = lps[k] + [float(logp[k, w])]
            if w == EOS or t == max_len:                       # O9 banking
                n = t
                bank.append((s / length_penalty(n, alpha), t, r, s, n_hyps[r], n_lps[r]))
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
    best = sorted(bank, key=lambda b: (-b[0], b[1], b[2]))[0]
    out = {"tokens": list(best[4]), "norm": best[0], "raw": best[3], "t": best[1], "r": best[2],
           "token_logp": list(best[5]), "bank": bank}
    if trace:
        out["steps"] = steps
    return out


def greedy(model: OracleModel, src: List[int], max_len: int) -> Dict:
    """O12: argmax with the lowest id on ties; stop at EOS or max_len."""
    memory, finals = model.encode(src)
    y, ht, st = model.init_decoder(finals, 1)
    toks, lps = [], []
    for t in range(1, max_len + 1):
        logp, _, ht, st = model.decode_step(y, ht, st, memory)
        w = int(np.argmax(logp[0]))          # np.argmax returns the first maximum
        toks.append(w); lps.append(float(logp[0, w]))
        y = np.array([w])
        if w == EOS:
            break
    return {"tokens": toks, "raw": float(np.sum(lps)), "token_logp": lps}


def score_sequence(model: OracleModel, src: List[int], Y: List[int]) -> List[float]:
    """Teacher-forced log p(y_t | y_<t, x) of every token of Y (P105-108)."""
    memory, finals = model.encode(src)
    y, ht, st = model.init_decoder(finals, 1)
    out = []
    for w in Y:
        logp, _, ht, st = model.decode_step(y, ht, st, memory)
        out.append(float(logp[0, w]))
        y = np.array([w])
    return out


def brute_force(model: OracleModel, src: List[int], max_len: int, alpha: float = 0.0) -> List[Dict]:
    """O12: enumerate Y = {sequences ending at their first EOS, length <= max_len}
    U {EOS-free sequences of length exactly max_len}; score each by teacher
    forcing.  Returns all of them sorted by (norm desc, then token tuple)."""
    V = model.V
    out = []
    for n in range(1, max_len + 1):
        for prefix in itertools.product([w for w in range(V) if w != EOS], repeat=n - 1):
            tails = [EOS] if n < max_len else list(range(V))
            for last in tails:
                Y = list(prefix) + [last]
                lp = score_sequence(model, src, Y)
                raw = float(np.sum(lp))
                out.append({"tokens": Y, "raw": raw, "norm": raw / length_penalty(n, alpha),
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
           "length_penalty", "unpad", "model_from_file", "Optional"]
