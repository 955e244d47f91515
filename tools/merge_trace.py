import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ONMT_MERGE_TRACE"] = "1"; os.environ["ONMT_USE_GRAPH"] = "0"
import synth, paper_1805_11462_b200 as ob
d = tempfile.mkdtemp()
m = ob.Model(synth.weights_file("c2", d), 0, "bf16")
ids, lens = synth.make_corpus("c2")
for i in range(3):
    m.translate(ids, lens, 5, 8, 0.0)
