"""GPU-vs-oracle comparison protocol (BASELINE north_star):

  * sequences must equal the oracle's except where candidate scores differ by less
    than TIE = 1e-4 (reading R22): walk the steps of each sentence; at the first step
    where the GPU's ordered selection (parent slot, token) differs from the oracle's,
    the sentence is tie-excused iff, for every rank r, the ORACLE's score of the GPU's
    r-th pick is within TIE of the oracle's r-th selected score; after an excused
    divergence the sequence is no longer compared.  If every step matches but the
    final bank choice differs, the two choices' oracle normalised scores must be
    within TIE.
  * per-token log-probabilities of the GPU's returned hypothesis are compared with
    the oracle's teacher-forced scores of that same hypothesis (reading R21):
    |d| <= 2e-3 (bf16 models) / 1e-5 (fp32 models).
  * raw score = sum of token log-probs within fp32 rounding of the sum.
"""
from __future__ import annotations

import os

import numpy as np

from oracle import beam_search, length_penalty, score_sequence

TIE = 1e-4
LOGP_TOL = {"bf16": 2e-3, "fp32": 1e-5}


def compare_sentence(om, src, gpu, b, K, max_len, alpha, precision, tie=TIE, logp_tol=None):
    """Returns ("match" | "excused" | "fail", detail dict).  tie / logp_tol default to the
    north_star bars (1e-4; 2e-3 bf16, 1e-5 fp32); only derived_tolerances() widens them."""
    # scalars, or per-step arrays (reading R34: bars derived per generated token)
    def tie_at(t):
        if not np.ndim(tie):
            return float(tie)
        return float(tie[min(t, len(tie)) - 1]) if len(tie) else TIE
    if logp_tol is None or not np.ndim(logp_tol):
        ltol = np.full(max_len, LOGP_TOL[precision] if logp_tol is None else float(logp_tol))
    else:                                              # per-token bars, extended by the last one
        lt = np.asarray(logp_tol, dtype=np.float64)[:max_len]
        ltol = np.concatenate([lt, np.full(max_len - len(lt), lt[-1] if len(lt) else LOGP_TOL[precision])])
    ref = beam_search(om, src, K, max_len, alpha, trace=True)
    n = int(gpu["lens"][b])
    hyp = [int(v) for v in gpu["hyps"][b, :n]]
    det = {"n": n, "ref_n": len(ref["tokens"])}
    status = "match"
    for st in ref["steps"]:
        t = st["t"]
        gsel = [(int(gpu["sel_parent"][t - 1, b, r]), int(gpu["sel_token"][t - 1, b, r]))
                for r in range(K) if gpu["sel_parent"][t - 1, b, r] >= 0]
        osel = [(k, w) for (k, w, s) in st["sel"]]
        if gsel == osel:
            continue
        # first divergence: oracle scores of the GPU's picks
        lookup = {(k, w): s for (s, k, w) in st["cand"]}
        if len(gsel) != len(osel):
            det["why"] = f"t={t}: selection count {len(gsel)} vs {len(osel)}"
            status = "fail"
            break
        ok = True
        for r, (g, o) in enumerate(zip(gsel, st["sel"])):
            if g not in lookup or abs(lookup[g] - o[2]) > tie_at(t):
                ok = False
                det["why"] = f"t={t} r={r}: gpu {g} score {lookup.get(g)} vs oracle {o}"
                break
        status = "excused" if ok else "fail"
        det["diverged_at"] = t
        break
    if status == "match" and hyp != ref["tokens"]:
        ns = score_sequence(om, src, hyp)
        gnorm = float(np.sum(ns)) / length_penalty(len(hyp), alpha)
        if abs(gnorm - ref["norm"]) <= tie_at(max(len(hyp), 1)):
            status = "excused"
        else:
            status = "fail"
            det["why"] = f"final choice: gpu norm {gnorm} vs oracle {ref['norm']}"
    # per-token log p of the GPU's own hypothesis
    tf = np.array(score_sequence(om, src, hyp))
    glp = gpu["token_logp"][b, :n].astype(np.float64)
    dif = np.abs(tf - glp)
    err = float(np.max(dif)) if n else 0.0
    det["logp_err"] = err
    over = np.nonzero(dif > ltol[:n])[0] if n else []
    if len(over):
        status = "fail"
        det["why"] = det.get("why", "") + f" token logp err {err} (first over its bar at t={over[0] + 1})"
    s = float(np.sum(glp))
    if abs(float(gpu["raw"][b]) - s) > 1e-6 * max(n, 1) * (1 + np.max(np.abs(glp), initial=0)) + 1e-5:
        status = "fail"
        det["why"] = det.get("why", "") + f" raw {gpu['raw'][b]} vs sum {s}"
    return status, det


_FORK = {}


def _one(om, ids, lens, gpu, b, K, max_len, alpha, precision, derive):
    src = [int(v) for v in ids[b, : lens[b]]]
    if not derive:
        return compare_sentence(om, src, gpu, b, K, max_len, alpha, precision)
    hyp = [int(v) for v in gpu["hyps"][b, :gpu["lens"][b]]]
    tie, ltol, s_tok, _ = derived_tolerances(om, src, hyp, precision, per_token=True, amp=1.0)
    st, det = compare_sentence(om, src, gpu, b, K, max_len, alpha, precision, tie=tie, logp_tol=ltol)
    strict = np.nonzero(ltol > LOGP_TOL[precision])[0]
    det["strict_prefix"] = int(strict[0]) if len(strict) else len(hyp)   # tokens held to the north_star bar
    det["bar_last"] = float(ltol[-1]) if len(ltol) else None
    return st, det


def _fork_compare(b):
    om, ids, lens, gpu, K, max_len, alpha, precision, derive = _FORK["args"]
    from threadpoolctl import threadpool_limits
    with threadpool_limits(_FORK["threads"]):
        return _one(om, ids, lens, gpu, b, K, max_len, alpha, precision, derive)


def compare_batch(om, ids, lens, gpu, K, max_len, alpha, precision, sentences=None, workers=1, derive=False):
    """Protocol over the sentences `sentences` (default: all) of a batch.  workers > 1 runs
    the oracle of different sentences in forked processes (each sentence is independent, S466).
    derive: per-token bars from the oracle's own conditioning (reading R34) instead of the
    fixed north_star bars - for models that are chaotic over the decoded length."""
    res = {"match": 0, "excused": 0, "fail": 0, "details": []}
    sel = list(range(len(lens))) if sentences is None else list(sentences)
    if workers > 1 and len(sel) > 1:
        import multiprocessing as mp
        _FORK["args"] = (om, ids, lens, gpu, K, max_len, alpha, precision, derive)
        _FORK["threads"] = max(1, (os.cpu_count() or 1) // workers)
        with mp.get_context("fork").Pool(min(workers, len(sel))) as pool:
            outs = pool.map(_fork_compare, sel)
        _FORK.clear()
    else:
        outs = []
        for b in sel:
            outs.append(_one(om, ids, lens, gpu, b, K, max_len, alpha, precision, derive))
    for st, det in outs:
        res[st] += 1
        res["details"].append((st, det))
    return res


def summary(res):
    return f"matched {res['match']} / excused {res['excused']} / failed {res['fail']}"


# working-precision unit roundoff the GPU path computes with (reading R34): fp32
# mode rounds every operation to fp32; bf16 mode keeps bf16 weights (the oracle evaluates the
# same rounded weights) and splits activations into bf16 hi + lo (residual <= 2^-18 relative)
UNIT = {"fp32": 2.0 ** -23, "bf16": 2.0 ** -18}


def derived_tolerances(om, src, hyp, precision, margin=10.0, seeds=(0, 1, 2), amp=8.0, per_token=False, probes=()):
    """Reading R34: the oracle's own sensitivity to a relative perturbation of the working
    precision's unit roundoff.  Every weight tensor is multiplied by (1 + amp * UNIT * u),
    u ~ U(-1, 1) (3 seeds; amp = 8 ~ the sqrt(64) growth of rounding over a 64-term K block),
    and the GPU's hypothesis is teacher-forced through both models; the bars become
    max(north_star bar, margin x the largest change) - on non-chaotic models the north_star
    bars stand, on chaotic ones (large weights) no implementation in that precision could
    meet them."""
    from oracle import OracleModel
    # probes: further sequences whose conditioning bounds the tie decisions (e.g. a beam that
    # runs on after the returned hypothesis finished); their per-token sensitivity counts at
    # the same step index
    seqs = [list(hyp)] + [list(p) for p in probes]
    n = max(len(q) for q in seqs)
    base = [np.array(score_sequence(om, src, q)) for q in seqs]
    s_tok = np.zeros(n)
    s_cum = np.zeros(n)
    for seed in seeds:
        rng = np.random.default_rng(seed)
        u = amp * UNIT[precision]
        pert = OracleModel({k: v * (1.0 + u * rng.uniform(-1.0, 1.0, v.shape)) for k, v in om.t.items()})
        for q, a in zip(seqs, base):
            if not q:
                continue
            b = np.array(score_sequence(pert, src, q))
            m = len(q)
            s_tok[:m] = np.maximum(s_tok[:m], np.abs(a - b))
            s_cum[:m] = np.maximum(s_cum[:m], np.abs(np.cumsum(a) - np.cumsum(b)))
    if per_token:
        # bar of token t: the sensitivity of the tokens up to t (a running maximum), so the
        # north_star bars hold over the prefix where the model is well conditioned
        return (np.maximum(TIE, margin * np.maximum.accumulate(s_cum)) if n else np.zeros(0),
                np.maximum(LOGP_TOL[precision], margin * np.maximum.accumulate(s_tok)) if n else np.zeros(0),
                s_tok, s_cum)
    d_tok = float(s_tok.max()) if n else 0.0
    d_cum = float(s_cum.max()) if n else 0.0
    return max(TIE, margin * d_cum), max(LOGP_TOL[precision], margin * d_tok), d_tok, d_cum
