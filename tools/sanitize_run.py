"""Small translations for compute-sanitizer runs (one tool per process): c1 (fp32, SIMT path),
a bf16 toy model through the tcgen05 path with one row group, and the same toy model with
two row groups (R = 300: the generator's non-overlapped plan)."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1805_11462_b200 as ob  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
with tempfile.TemporaryDirectory() as d:
    if which in ("all", "c1"):
        path = synth.weights_file("c1", d)
        ids, lens = synth.make_corpus("c1")
        with ob.Model(path, 0, "fp32") as m:
            m.set_option("use_graph", 0)
            out = m.translate(ids, lens, 3, 10, 0.0)
        print("c1", out["lens"].tolist(), flush=True)
    if which in ("all", "toy"):
        cfg = synth.ModelConfig(2, 64, 128, 300, 50000, False, True)
        p2 = os.path.join(d, "toy.mnmt")
        synth.write_mnmt(p2, synth.random_model_tensors(cfg, 3, 0.1))
        rng = np.random.default_rng(0)
        with ob.Model(p2, 0, "bf16") as m:
            m.set_option("use_graph", 0)
            for B in (6, 60):
                lens = rng.integers(3, 12, B).astype(np.int32)
                ids = np.zeros((B, 12), np.int32)
                for b in range(B):
                    ids[b, :lens[b]] = rng.integers(4, 300, lens[b])
                out = m.translate(ids, lens, 5, 3, 0.0)
                print("toy B", B, out["lens"][:4].tolist(), flush=True)
