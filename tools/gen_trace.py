"""Timeline of the persistent generator kernel on the c2 model (ONMT_GEN_TRACE=1)."""
import os, sys, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1805_11462_b200 as ob
d = tempfile.mkdtemp()
path = synth.weights_file("c2", d)
m = ob.Model(path, 0, "bf16")
h = np.tanh(np.random.default_rng(0).normal(size=(150, 500))).astype(np.float32)
for i in range(3):
    m.test_gen(h, 5)
os.environ["ONMT_GEN_TRACE"] = "1"
m.test_gen(h, 5)
