"""Experiment: two half-batch decode chains on two streams, each sized for half the SMs
(ONMT_NUM_SMS), against one full-batch chain on the whole GPU (c2 workload)."""
import os, sys, tempfile, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1805_11462_b200 as ob

d = os.environ.get("ONMT_WEIGHT_CACHE", tempfile.mkdtemp())
path = synth.weights_file("c2", d)
ids, lens = synth.make_corpus("c2")
dev = torch.device("cuda", 0)
K, ML = 5, 100


def mk(nsm, ids_np, lens_np, stream):
    if nsm:
        os.environ["ONMT_NUM_SMS"] = str(nsm)
    else:
        os.environ.pop("ONMT_NUM_SMS", None)
    m = ob.Model(path, 0, "bf16")
    m.set_stream(stream.cuda_stream)
    B = len(lens_np)
    with torch.cuda.stream(stream):
        i_d = torch.from_numpy(np.ascontiguousarray(ids_np)).to(dev)
        l_d = torch.from_numpy(np.ascontiguousarray(lens_np)).to(dev)
        out = {"hyps": torch.zeros((B, ML), dtype=torch.int32, device=dev),
               "lens": torch.zeros(B, dtype=torch.int32, device=dev),
               "scores": torch.zeros(B, dtype=torch.float32, device=dev),
               "raw": torch.zeros(B, dtype=torch.float32, device=dev),
               "token_logp": torch.zeros((B, ML), dtype=torch.float32, device=dev)}
    return m, (i_d, l_d, out, lens_np)


def run(m, a):
    m.translate_dev(a[0], a[1], K, ML, 0.0, a[2], a[3])


main = torch.cuda.current_stream()
s0, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
S = int(lens.max())
full, fa = mk(None, ids[:, :S], lens, s0)
h = len(lens) // 2
A, aa = mk(int(os.environ.get("HALF_SMS", "74")), ids[:h, :S], lens[:h], s1)
Bm, ba = mk(int(os.environ.get("HALF_SMS", "74")), ids[h:, :S], lens[h:], s2)
for _ in range(3):
    run(full, fa); run(A, aa); run(Bm, ba)
torch.cuda.synchronize()
reps = 10
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(s0)
for _ in range(reps):
    run(full, fa)
t1.record(s0)
torch.cuda.synchronize()
full_ms = t0.elapsed_time(t1) / reps
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(); e3 = torch.cuda.Event()
e0.record(main)
s1.wait_event(e0); s2.wait_event(e0)
for _ in range(reps):
    run(A, aa); run(Bm, ba)
e2.record(s1); e3.record(s2)
main.wait_event(e2); main.wait_event(e3)
e1.record(main)
torch.cuda.synchronize()
dual_ms = e0.elapsed_time(e1) / reps
tok_full = int(fa[2]["lens"].sum()); tok_dual = int(aa[2]["lens"].sum()) + int(ba[2]["lens"].sum())
print(f"full: {full_ms:.3f} ms/call  {tok_full / full_ms * 1e3:.0f} tok/s")
print(f"dual: {dual_ms:.3f} ms/call  {tok_dual / dual_ms * 1e3:.0f} tok/s")
same = torch.equal(torch.cat([aa[2]['hyps'], ba[2]['hyps']]), fa[2]['hyps'])
print("dual hyps == full hyps:", same)
