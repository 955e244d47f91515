"""Per-CTA phase stamps of the fused decoder step (library built with EXTRA=-DONMT_KTRACE):
runs a short c2 translation without the CUDA graph and prints the last step's timeline."""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ONMT_USE_GRAPH"] = "0"
import synth, paper_1805_11462_b200 as ob
d = os.environ.get("ONMT_WEIGHT_CACHE", tempfile.mkdtemp())
m = ob.Model(synth.weights_file("c2", d), 0, "bf16")
ids, lens = synth.make_corpus("c2")
m.translate(ids, lens, 5, 6, 0.0)
os.environ["ONMT_PHASES"] = "1"
m.translate(ids, lens, 5, 6, 0.0)
