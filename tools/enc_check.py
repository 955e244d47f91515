import os, sys, tempfile, numpy as np
sys.path.insert(0, os.getcwd())
import synth, paper_1805_11462_b200 as ob
for wl in ["c2", "c3"]:
    d = tempfile.mkdtemp()
    path = synth.weights_file(wl, d)
    ids, lens = synth.make_corpus(wl)
    ids, lens = ids[:30], lens[:30]
    S = int(lens.max()); ids = np.ascontiguousarray(ids[:, :S])
    outs = {}
    for pers in (0, 1):
        os.environ["ONMT_ENC_PERSISTENT"] = str(pers)
        m = ob.Model(path, 0, "bf16")
        mem, h, c = m.encode(ids, lens)
        o = m.translate(ids, lens, 5, 20, 0.0)
        outs[pers] = (mem, h, c, o)
    a, b = outs[0], outs[1]
    print(wl, "mem maxdiff", np.abs(a[0] - b[0]).max(), "h", np.abs(a[1] - b[1]).max(), "c", np.abs(a[2] - b[2]).max(),
          "hyps equal", np.array_equal(a[3]["hyps"], b[3]["hyps"]))
