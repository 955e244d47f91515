"""Diagnostic: token log-p error vs the oracle for the first sentences of a workload's batch,
per batch size and per runtime option (localises a multi-row-group bug)."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1805_11462_b200 as ob  # noqa: E402
from oracle import OracleModel, load_model_tensors, score_sequence  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
ML = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
path = synth.weights_file(wl, cache)
w = synth.WORKLOADS[wl]
om = OracleModel(load_model_tensors(path, "bf16"))
ids_all, lens_all = synth.make_corpus(wl)
m = ob.Model(path, 0, "bf16")
ref = {}
Bs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [8, 48, 52, 64]
for B in Bs:
    for opt in ([], [("fold_wout", 0)], [("fused_gemm", 0)], [("gen_step", 0)]):
        for k, v in opt:
            m.set_option(k, v)
        ids, lens = ids_all[:B], lens_all[:B]
        S = int(lens.max())
        out = m.translate(np.ascontiguousarray(ids[:, :S]), lens, w.decode.beam, ML, w.decode.alpha)
        errs = []
        for b in (0, B - 1):
            src = [int(x) for x in ids[b, :lens[b]]]
            hyp = [int(x) for x in out["hyps"][b, :out["lens"][b]]]
            tf = np.array(score_sequence(om, src, hyp))
            errs.append(float(np.max(np.abs(tf - out["token_logp"][b, :len(hyp)]))))
        print(f"{wl} B={B} R={B * w.decode.beam} opts={opt}: max token logp err sent0 {errs[0]:.2e} sent{B-1} {errs[1]:.2e}",
              flush=True)
        for k, v in opt:
            m.set_option(k, 1)
