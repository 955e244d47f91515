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
    TIE_ = tie
    LTOL = LOGP_TOL[precision] if logp_tol is None else logp_tol
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
            if g not in lookup or abs(lookup[g] - o[2]) > TIE_:
                ok = False
                det["why"] = f"t={t} r={r}: gpu {g} score {lookup.get(g)} vs oracle {o}"
                break
        status = "excused" if ok else "fail"
        det["diverged_at"] = t
        break
    if status == "match" and hyp != ref["tokens"]:
        ns = score_sequence(om, src, hyp)
        gnorm = float(np.sum(ns)) / length_penalty(len(hyp), alpha)
        if abs(gnorm - ref["norm"]) <= TIE_:
            status = "excused"
        else:
            status = "fail"
            det["why"] = f"final choice: gpu norm {gnorm} vs oracle {ref['norm']}"
    # per-token log p of the GPU's own hypothesis
    tf = np.array(score_sequence(om, src, hyp))
    glp = gpu["token_logp"][b, :n].astype(np.float64)
    err = float(np.max(np.abs(tf - glp))) if n else 0.0
    det["logp_err"] = err
    if err > LTOL:
        status = "fail"
        det["why"] = det.get("why", "") + f" token logp err {err}"
    s = float(np.sum(glp))
    if abs(float(gpu["raw"][b]) - s) > 1e-6 * max(n, 1) * (1 + np.max(np.abs(glp), initial=0)) + 1e-5:
        status = "fail"
        det["why"] = det.get("why", "") + f" raw {gpu['raw'][b]} vs sum {s}"
    return status, det


_FORK = {}


def _fork_compare(b):
    om, ids, lens, gpu, K, max_len, alpha, precision = _FORK["args"]
    from threadpoolctl import threadpool_limits
    with threadpool_limits(_FORK["threads"]):
        src = [int(v) for v in ids[b, : lens[b]]]
        return compare_sentence(om, src, gpu, b, K, max_len, alpha, precision)


def compare_batch(om, ids, lens, gpu, K, max_len, alpha, precision, sentences=None, workers=1):
    """Protocol over the sentences `sentences` (default: all) of a batch.  workers > 1 runs
    the oracle of different sentences in forked processes (each sentence is independent, S466)."""
    res = {"match": 0, "excused": 0, "fail": 0, "details": []}
    sel = list(range(len(lens))) if sentences is None else list(sentences)
    if workers > 1 and len(sel) > 1:
        import multiprocessing as mp
        _FORK["args"] = (om, ids, lens, gpu, K, max_len, alpha, precision)
        _FORK["threads"] = max(1, (os.cpu_count() or 1) // workers)
        with mp.get_context("fork").Pool(min(workers, len(sel))) as pool:
            outs = pool.map(_fork_compare, sel)
        _FORK.clear()
    else:
        outs = []
        for b in sel:
            src = [int(v) for v in ids[b, : lens[b]]]
            outs.append(compare_sentence(om, src, gpu, b, K, max_len, alpha, precision))
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


def derived_tolerances(om, src, hyp, precision, margin=10.0, seed=0):
    """Reading R34: the oracle's own sensitivity to a relative perturbation of the working
    precision's unit roundoff.  Every weight tensor is multiplied by (1 + UNIT * u), u ~ U(-1, 1)
    seeded, and the GPU's hypothesis is teacher-forced through both models; the bars become
    max(north_star bar, margin x the measured change) - on non-chaotic models the north_star
    bars stand, on chaotic ones (large weights) no implementation in that precision could
    meet them."""
    from oracle import OracleModel
    rng = np.random.default_rng(seed)
    pert = OracleModel({k: v * (1.0 + UNIT[precision] * rng.uniform(-1.0, 1.0, v.shape)) for k, v in om.t.items()})
    a = np.array(score_sequence(om, src, hyp))
    b = np.array(score_sequence(pert, src, hyp))
    d_tok = float(np.max(np.abs(a - b))) if len(hyp) else 0.0
    d_cum = float(np.max(np.abs(np.cumsum(a) - np.cumsum(b)))) if len(hyp) else 0.0
    return max(TIE, margin * d_cum), max(LOGP_TOL[precision], margin * d_tok), d_tok, d_cum
