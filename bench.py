"""Benchmark: batched beam-5 translation (BASELINE.json metric) on synthetic c2 inputs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A "step" is one pass of the whole hot path (encoder + every decode step + beam
bookkeeping + finalize, DESIGN.md §2 A1-A11) over one batch of synthetic input, through
the C-ABI (onmt_translate_dev: inputs already resident in HBM).  `e2e` re-measures the
same metric through the host-buffer C-ABI call (onmt_translate), H2D/D2H copies inside
the timed region.  Multi-GPU (torchrun, one process per GPU): every rank translates its
own fixed-size batch from one seeded corpus (weak scaling), then hypotheses are
all-gathered over NCCL (the only collective of the path); time is the max
over ranks of the device-timed steps.  L2 is flushed (a 512 MB write) between timed
steps.  `--impl reference` times the fp64 CPU oracle on a bounded sample instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def peaks():
    if os.path.exists(PEAKS_PATH):
        p = json.load(open(PEAKS_PATH))
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            t0 = time.time()                    # the sampler is live (first row written) before timing
            while time.time() - t0 < 5.0 and os.path.getsize(self.f.name) == 0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.skip = len(open(self.f.name).read().strip().splitlines())   # rows from before timing
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines()[getattr(self, "skip", 0):] if l.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


FAMILIES = ["gen", "step", "encode", "gemm", "cell", "attention", "attn_out", "merge"]


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def gen_roofline_terms(w: synth.Workload, R: int, gate_tiles: int = 0):
    """Algorithmic bytes / flops of ONE generator launch:
    bytes = 2*H*V (bf16 W_gen) + 4*V (fp32 bias); flops = 2*R*H*V.  With the recurrent-split
    step the same launch also computes the next step's recurrent gate terms:
    + 2*(L+1)*4H*H weight bytes and 2*R*(L+1)*4H*H flops (W_feed and every layer's W_hh)."""
    H, V, L = w.model.hidden, w.model.v_tgt, w.model.layers
    b, f = 2.0 * H * V + 4.0 * V, 2.0 * R * H * V
    if gate_tiles:
        b += 2.0 * (L + 1) * 4 * H * H
        f += 2.0 * R * (L + 1) * 4 * H * H
    return b, f


# ---------------------------------------------------------------------------- ours
def corpus_run(model, args, w, ws, rank, dev):
    """Corpus mode (SURVEY §8(d) timing corpus; PAPER.md P233-235 "translating a large set of
    sentences"): the workload's corpus (c2: 30 x 8 x 16 = 3840 sentences) cut into batches of
    the workload's size in corpus order, dealt round-robin to the ranks, each batch trimmed to
    its own longest source and translated through the host API (onmt_translate: H2D of its
    ids / lengths and D2H of every output inside the timed region), then one gather of every
    output with the original indices.  Whole-corpus tokens / the max over ranks of the wall
    time of the (barrier-bracketed) pass; one untimed pass first captures the few graphs the
    bucketed source lengths need."""
    import torch
    import torch.distributed as dist
    from paper_1805_11462_b200.parallel import deal_batches, gather_results, make_batches, translate_batches
    B, K, ML, alpha = w.data.batch, w.decode.beam, w.decode.max_len, w.decode.alpha
    n = args.corpus_sentences or CORPUS[args.workload]
    ids, lens = synth.make_corpus(args.workload, n)
    batches = make_batches(n, B)
    mine = deal_batches(len(batches), ws, rank)
    model.set_stream(None)
    translate_batches(model, ids, lens, batches, mine, K, ML, alpha)      # warm-up: graphs captured
    cap0 = model.graph_captures()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    local, idx = translate_batches(model, ids, lens, batches, mine, K, ML, alpha)
    if ws > 1:
        g = gather_results({k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in local.items()},
                           torch.from_numpy(idx).to(dev), n_total=n)
        total_tokens = int(g["lens"].sum().item())
    else:
        total_tokens = int(local["lens"].sum())
    dt = time.perf_counter() - t0
    recaptures = model.graph_captures() - cap0
    if ws > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": round(total_tokens / dt, 1), "unit": "target tok/s", "sentences": n, "batches": len(batches),
            "batch": B, "tokens": total_tokens, "wall_s": round(dt, 4), "graph_captures_in_timed_pass": int(recaptures),
            "graphs_cached": int(cap0), "timing": "host wall clock, barrier-bracketed, max over ranks; host API "
            "(H2D/D2H per batch inside); batches dealt round-robin, one gather of every output + indices"}


# default corpus sizes (bounded so a default run ends in minutes); SURVEY §8(d)'s full c4 corpus is
# --corpus-sentences 16384
CORPUS = {"c1": 2, "c2": 3840, "c3": 64 * 8, "c4": 128 * 8, "c5": 16 * 8}


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1805_11462_b200 as ob

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = synth.WORKLOADS[args.workload]
    B_wl, K, ML, alpha = w.data.batch, w.decode.beam, w.decode.max_len, w.decode.alpha
    cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
    if rank == 0 or ws == 1:
        path = synth.weights_file(args.workload, cache)
    if ws > 1:
        dist.barrier()
        path = synth.weights_file(args.workload, cache)
    model = ob.Model(path, local, w.decode.precision)
    from paper_1805_11462_b200.parallel import gather_results, rank_slice
    if args.vocab_parallel:
        # vocabulary-parallel generator: every rank decodes the SAME batch and
        # streams 1/world of W_gen; partials are exchanged through peer memory inside the graph
        ids_all, lens_all = synth.make_corpus(args.workload)
        b0, b1 = 0, B_wl
    elif args.scaling == "weak":
        # weak scaling: rank r translates its own full batch, sentences [r*B, (r+1)*B) of one corpus
        ids_all, lens_all = synth.make_corpus(args.workload, B_wl * ws)
        b0, b1 = rank_slice(B_wl * ws, ws, rank)
    else:
        # strong scaling: the workload's one batch sharded by sentence over the ranks
        ids_all, lens_all = synth.make_corpus(args.workload)
        b0, b1 = rank_slice(B_wl, ws, rank)
    B = b1 - b0
    ids = np.ascontiguousarray(ids_all[b0:b1])
    lens = np.ascontiguousarray(lens_all[b0:b1])
    S = int(lens.max())
    ids = np.ascontiguousarray(ids[:, :S])
    if args.vocab_parallel:
        from paper_1805_11462_b200.parallel import open_vocab_parallel
        model.set_option("rsplit", 0)
        if ws > 1:
            open_vocab_parallel(model, (b1 - b0) * K)
        else:
            model.vp_handle((b1 - b0) * K)
            model.vp_open(1, 0, None)
    stream = torch.cuda.Stream(device=dev)
    model.set_stream(stream.cuda_stream)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    with torch.cuda.stream(stream):
        ids_d = torch.from_numpy(ids).to(dev)
        lens_d = torch.from_numpy(lens).to(dev)
        index_d = torch.arange(b0, b1, dtype=torch.int64, device=dev)
        out = {"hyps": torch.zeros((B, ML), dtype=torch.int32, device=dev),
               "lens": torch.zeros(B, dtype=torch.int32, device=dev),
               "scores": torch.zeros(B, dtype=torch.float32, device=dev),
               "raw": torch.zeros(B, dtype=torch.float32, device=dev),
               "token_logp": torch.zeros((B, ML), dtype=torch.float32, device=dev)}

    def step():
        model.translate_dev(ids_d, lens_d, K, ML, alpha, out, lens)
        if ws > 1 and not args.vocab_parallel:
            gather_results(out, index_d)        # the path's only collective (NCCL all-gather)

    def timed_pass(profile):
        model.set_option("profile", profile)
        step()                                  # (re)capture this variant's graph outside timing
        stream.synchronize()
        model.launches(reset=True)
        for fam in FAMILIES:
            model.kernel_time(fam, reset=True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()                       # L2 flush between timed steps
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        return sum(a.elapsed_time(b) for a, b in evs), model.launches(reset=True)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        stream.synchronize()
        # (1) THE timed region: uninstrumented graph (no event nodes between kernels)
        model.set_option("profile", 0)
        step()
        stream.synchronize()
        clk = ClockSampler(local)
        clk.start()
        t_ms, launches = timed_pass(0)
        clocks = clk.stop()
        tokens = int(out["lens"].sum().item()) * args.steps
        # (2) same steps again with CUDA events around every generator launch (the roofline's
        #     per-launch duration; the events serialise the generator with its neighbours)
        t_ms_gen_pass, _ = timed_pass(1)
        gen_ms, gen_n = model.kernel_time("gen", reset=True)
        # (3) one untimed call with every kernel family instrumented, for the breakdown
        model.set_option("profile", 2)
        step()
        stream.synchronize()
        for fam in FAMILIES:
            model.kernel_time(fam, reset=True)
        step()
        fam_t = {fam: model.kernel_time(fam, reset=True) for fam in FAMILIES}
        model.set_option("profile", 0)
    if ws > 1:
        tt = torch.tensor([t_ms, float(tokens)], dtype=torch.float64, device=dev)
        tmax = tt.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        if not args.vocab_parallel:            # (vocabulary-parallel: every rank decodes the same batch)
            dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        t_ms, tokens = float(tmax[0].item()), int(tt[1].item())
        if args.vocab_parallel:                 # every rank must hold the same translation
            g = torch.empty((ws,) + tuple(out["hyps"].shape), dtype=out["hyps"].dtype, device=dev)
            dist.all_gather_into_tensor(g, out["hyps"].contiguous())
            assert bool((g == g[:1]).all().item()), "vocabulary-parallel ranks disagree"
    value = tokens / (t_ms / 1e3)

    # ---- e2e: host buffers through onmt_translate, H2D / D2H inside the timed region
    model.set_stream(None)
    model.translate(ids, lens, K, ML, alpha)        # warm-up: capture the host-API graph untimed
    e2e_ms = []
    if ws > 1:
        dist.barrier()
    for i in range(max(1, args.steps)):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = model.translate(ids, lens, K, ML, alpha)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_tokens = int(r["lens"].sum()) * len(e2e_ms)
    e2e_t = sum(e2e_ms)
    if ws > 1:
        tt = torch.tensor([e2e_t, float(e2e_tokens)], dtype=torch.float64, device=dev)
        tm = tt.clone()
        dist.all_reduce(tm[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        e2e_t, e2e_tokens = float(tm[0].item()), int(tt[1].item())
    h2d = ids.nbytes + lens.nbytes
    d2h = B * ML * 4 * 2 + B * 4 * 3
    model_plan = model.last_plan()
    corpus = corpus_run(model, args, w, ws, rank, dev) if not (args.no_corpus or args.vocab_parallel) else None

    if rank == 0:
        pk = peaks()
        R = B * K
        plan = model_plan
        gbytes, gflops = gen_roofline_terms(w, R, plan.get("gate_tiles", 0))
        gen_avg_s = (gen_ms / gen_n) / 1e3 if gen_n else float("nan")
        achieved = gbytes / gen_avg_s / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"gen_traffic_{args.workload}.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "target tok/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong" if args.vocab_parallel else args.scaling,
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded U(-0.1,0.1) weights, Zipf(1.1) ids; DESIGN.md §3)",
            "config": {"workload": args.workload, "model": "2x500 LSTM enc-dec, general attn, input feed, V=50k"
                       if args.workload == "c2" else args.workload,
                       "global_batch": B_wl * ws if args.scaling == "weak" else B_wl, "batch_per_gpu": B,
                       "beam": K, "max_len": ML,
                       "length_penalty": alpha, "src_len": [w.data.len_lo, w.data.len_hi],
                       "parallelism": (f"vocab-parallel generator over {ws} GPUs (peer-memory partial exchange)"
                                       if args.vocab_parallel else
                                       f"dp{ws} (sentence-sharded, NCCL all-gather of every output + indices)"),
                       "l2": "flushed (512 MB write) between timed steps; weights stay L2-resident "
                             "across the decode steps of one step",
                       "timed_graph": "uninstrumented (no CUDA-event nodes inside the call)"},
            "e2e": {"value": round(e2e_tokens / (e2e_t / 1e3), 1), "unit": "target tok/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "plan": model_plan,
            "roofline": {"kernel": "gen_step_kernel (K-outer tcgen05 generator + log-softmax + per-CTA top-K; logits never in HBM)",
                         "bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
                         "peak_src": pk["src"],
                         "algorithmic_bytes_per_launch": gbytes, "flops_per_launch": gflops,
                         "avg_launch_us": round(gen_avg_s * 1e6, 3), "launches": gen_n,
                         "timing": "CUDA events around every generator launch in a second timed pass of the "
                                   "same steps (ms_per_step of that pass: %.4f)" % (t_ms_gen_pass / args.steps),
                         "tensor_tflops_algorithmic": round(gflops / gen_avg_s / 1e12, 1),
                         "gen_share_of_step": round(gen_ms / t_ms_gen_pass, 4) if t_ms_gen_pass else None},
            "breakdown_profiled_pass": {
                "note": "one extra untimed call with CUDA events around every kernel family (events add a few "
                        "us per kernel)",
                "encode_ms": round(fam_t["encode"][0], 4),
                "decode_step_avg_us": round(1e3 * fam_t["step"][0] / max(fam_t["step"][1], 1), 3),
                "per_decode_step_us": {fam: round(1e3 * fam_t[fam][0] / max(fam_t["step"][1], 1), 3)
                                       for fam in FAMILIES if fam not in ("step", "encode")}},
            "clocks": clocks,
            "tokens_per_step": tokens // args.steps,
        }
        if corpus is not None:
            line["corpus"] = corpus
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.workload, path, args.cpu_sample_sentences)
        print(json.dumps(line), flush=True)
    model.close()
    if ws > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- oracle
def oracle_cores():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(th)) if th else 1
    except Exception:
        return 1


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _oracle_sample(om, w, ids, lens, n_sent, budget_s):
    from oracle import beam_search
    t0 = time.perf_counter()
    toks, done = 0, 0
    for b in range(min(n_sent, len(lens))):
        r = beam_search(om, [int(v) for v in ids[b, :lens[b]]], w.decode.beam, w.decode.max_len, w.decode.alpha)
        toks += len(r["tokens"])
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return toks, done, time.perf_counter() - t0


def cpu_baseline(workload: str, path: str, n_sent: int, budget_s: float = 20.0):
    """The fp64 oracle (as it stands) on a bounded sample of the same workload: the first
    sentences of the batch, each translated in full (beam, max_len as the workload), until
    n_sent sentences or ~budget_s seconds of CPU work - with the BLAS pool at all host cores
    (the reported value) and again at 1 thread (SURVEY §8(d) oracle timing, settings ii / i)."""
    from threadpoolctl import threadpool_limits
    from oracle import OracleModel, load_model_tensors
    w = synth.WORKLOADS[workload]
    om = OracleModel(load_model_tensors(path, w.decode.precision))
    ids, lens = synth.make_corpus(workload)
    toks, done, dt = _oracle_sample(om, w, ids, lens, n_sent, budget_s)
    with threadpool_limits(1):
        t1, d1, s1 = _oracle_sample(om, w, ids, lens, n_sent, budget_s / 2)
    return {"value": round(toks / dt, 3), "unit": "target tok/s", "cores": oracle_cores(), "kind": "oracle",
            "sample": f"first {done} sentences of the {workload} batch, full decode (beam {w.decode.beam}, "
                      f"max_len {w.decode.max_len}), fp64 numpy per sentence, {dt:.1f} s",
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model(),
            "single_thread": {"value": round(t1 / s1, 3), "cores": 1,
                              "sample": f"first {d1} sentences, BLAS pool limited to 1 thread, {s1:.1f} s"}}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    w = synth.WORKLOADS[args.workload]
    cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
    path = synth.weights_file(args.workload, cache)
    from oracle import OracleModel, beam_search, load_model_tensors
    om = OracleModel(load_model_tensors(path, w.decode.precision))
    ids, lens = synth.make_corpus(args.workload)
    src = [int(v) for v in ids[0, :lens[0]]]
    per = w.decode.max_len
    for _ in range(args.warmup):
        beam_search(om, src, w.decode.beam, 2, w.decode.alpha)
    t0 = time.perf_counter()
    toks = 0
    for i in range(args.steps):                 # one step = one sentence of the batch, full decode
        r = beam_search(om, [int(v) for v in ids[i % len(lens), :lens[i % len(lens)]]], w.decode.beam, per,
                        w.decode.alpha)
        toks += len(r["tokens"])
    dt = time.perf_counter() - t0
    v = toks / dt
    cores = oracle_cores()
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "target tok/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "beam": w.decode.beam, "max_len": per,
                       "sample": "1 sentence of the batch per step (fp64 oracle on host cores)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "target tok/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"per step: 1 sentence of the {args.workload} batch, full decode to max_len {per}"},
            "e2e": {"value": round(v, 3), "unit": "target tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_score(args):
    """Secondary workload: teacher-forced scoring of synthetic target
    sentences (Zipf ids, lengths uniform in [10, max_len]) for the workload's batch, through
    onmt_score (host buffers: H2D/D2H inside the timed region, so value == e2e).  Metric:
    target tokens scored per second."""
    import torch
    import paper_1805_11462_b200 as ob
    w = synth.WORKLOADS[args.workload]
    B, T = w.data.batch, w.decode.max_len
    cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
    path = synth.weights_file(args.workload, cache)
    model = ob.Model(path, 0, w.decode.precision)
    ids, lens = synth.make_corpus(args.workload)
    S = int(lens.max())
    ids = np.ascontiguousarray(ids[:, :S])
    rng = np.random.default_rng(7)
    tl = rng.integers(10, T + 1, B).astype(np.int32)
    ranks = np.arange(1, model.info["v_tgt"] - 3, dtype=np.float64)
    pz = ranks ** -1.1
    pz /= pz.sum()
    tgt = np.zeros((B, T), np.int32)
    for b in range(B):
        tgt[b, :tl[b]] = 3 + rng.choice(len(ranks), tl[b], p=pz) + 1
    for _ in range(args.warmup):
        model.score(ids, lens, tgt, tl)
    model.set_option("profile", 1)
    model.score(ids, lens, tgt, tl)
    model.kernel_time("gen", reset=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        model.score(ids, lens, tgt, tl)
    dt = time.perf_counter() - t0
    gen_ms, gen_n = model.kernel_time("gen", reset=True)
    model.set_option("profile", 0)
    toks = int(tl.sum()) * args.steps
    pk = peaks()
    H, V = model.info["hidden"], model.info["v_tgt"]
    rows = B * T
    flops = 2.0 * rows * H * V                              # algorithmic (hi/lo split not counted)
    gen_s = gen_ms / max(gen_n, 1) / 1e3
    line = {"metric": "target tokens/sec scored (teacher-forced NLL, SURVEY §8(f) rank 1)",
            "value": round(toks / dt, 1), "unit": "target tok/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if w.decode.precision == "bf16" else "f32",
            "data": "synthetic (Zipf(1.1) target ids, lengths U[10, max_len])",
            "config": {"workload": args.workload, "task": "score", "batch": B, "t_max": T},
            "e2e": {"value": round(toks / dt, 1), "unit": "target tok/s", "h2d_bytes_per_step": int(ids.nbytes + tgt.nbytes),
                    "d2h_bytes_per_step": int(B * T * 4)},
            "roofline": {"kernel": "tc_gemm_kernel<MODE_GEN> over every (step, sentence) row (log-softmax + gold gather)",
                         "bound": "tensor", "achieved": round(flops / gen_s / 1e12, 1),
                         "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                         "frac": round(flops / gen_s / 1e12 / pk["bf16_tflops"], 4), "traffic": None,
                         "avg_launch_us": round(gen_s * 1e6, 2), "flops_per_launch": flops}}
    print(json.dumps(line), flush=True)
    model.close()


def run_translate_ex(args):
    """Translation customisations on the workload's batch through
    onmt_translate_ex (host buffers: H2D/D2H inside the timed region, so value == e2e):
    GNMT coverage penalty beta = 0.2, 5-best lists, attention-based <unk> replacement.
    The same call with the customisations off is timed beside it (their overhead)."""
    import torch
    import paper_1805_11462_b200 as ob
    w = synth.WORKLOADS[args.workload]
    K, ML, alpha = w.decode.beam, w.decode.max_len, w.decode.alpha
    cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
    path = synth.weights_file(args.workload, cache)
    model = ob.Model(path, 0, w.decode.precision)
    ids, lens = synth.make_corpus(args.workload)
    S = int(lens.max())
    ids = np.ascontiguousarray(ids[:, :S])

    def timed(beta, nb, unk):
        for _ in range(args.warmup):
            model.translate_ex(ids, lens, K, ML, alpha, beta, nb, unk)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        toks = 0
        for _ in range(args.steps):
            r = model.translate_ex(ids, lens, K, ML, alpha, beta, nb, unk)
            toks += int(r["lens"][:, 0].sum())
        return toks / (time.perf_counter() - t0), r

    v_ext, r = timed(0.2, K, True)
    v_plain, _ = timed(0.0, 1, False)
    B = len(lens)
    line = {"metric": "target tokens/sec (1-best tokens), beam-5 translate with coverage penalty + n-best + "
                      "unk replacement (SURVEY §8(f) rank 2)",
            "value": round(v_ext, 1), "unit": "target tok/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (DESIGN.md §3)",
            "config": {"workload": args.workload, "task": "translate_ex", "batch": B, "beam": K, "max_len": ML,
                       "coverage_penalty": 0.2, "n_best": K, "replace_unk": True},
            "e2e": {"value": round(v_ext, 1), "unit": "target tok/s", "h2d_bytes_per_step": int(ids.nbytes + lens.nbytes),
                    "d2h_bytes_per_step": int(B * K * (ML * 4 * 3 + 4 * 3))},
            "same_call_plain": {"value": round(v_plain, 1), "note": "onmt_translate_ex with beta = 0, n_best = 1, "
                                                                   "no replacement (host API)"},
            "unk_emitted": int((r["hyps"][:, 0] == 1).sum())}
    print(json.dumps(line), flush=True)
    model.close()


def run_copy(args):
    """Copy / pointer generator on the workload's batch through
    onmt_translate_copy (host buffers, so value == e2e): the workload's model plus the copy
    gate (copy.w, copy.b; seeded like every weight), the synthetic dynamic dictionary of
    synth.make_src_ext.  The plain model's host call is timed beside it."""
    import dataclasses
    import torch
    import paper_1805_11462_b200 as ob
    w = synth.WORKLOADS[args.workload]
    K, ML, alpha = w.decode.beam, w.decode.max_len, w.decode.alpha
    cache = os.environ.get("ONMT_WEIGHT_CACHE", os.path.join(tempfile.gettempdir(), "onmt_weights"))
    os.makedirs(cache, exist_ok=True)
    cfg = dataclasses.replace(w.model, copy=True)
    path = os.path.join(cache, f"{args.workload}_copy_s{w.weight_seed}.mnmt")
    if not os.path.exists(path):
        synth.write_mnmt(path, synth.make_weights(cfg, w.weight_seed))
    model = ob.Model(path, 0, w.decode.precision)
    ids, lens = synth.make_corpus(args.workload)
    S = int(lens.max())
    ids = np.ascontiguousarray(ids[:, :S])
    ext = synth.make_src_ext(ids, lens, cfg.v_tgt)
    for _ in range(args.warmup):
        r = model.translate_copy(ids, lens, ext, K, ML, alpha)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    toks = 0
    for _ in range(args.steps):
        r = model.translate_copy(ids, lens, ext, K, ML, alpha)
        toks += int(r["lens"].sum())
    v = toks / (time.perf_counter() - t0)
    model.close()
    plain = ob.Model(synth.weights_file(args.workload, cache), 0, w.decode.precision)
    for _ in range(args.warmup):
        plain.translate(ids, lens, K, ML, alpha)
    t0 = time.perf_counter()
    pt = 0
    for _ in range(args.steps):
        pt += int(plain.translate(ids, lens, K, ML, alpha)["lens"].sum())
    vp = pt / (time.perf_counter() - t0)
    plain.close()
    B = len(lens)
    line = {"metric": "target tokens/sec, beam translate of a copy / pointer-generator model over the extended "
                      "vocabulary (SURVEY §8(f) rank 3)",
            "value": round(v, 1), "unit": "target tok/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": w.decode.precision.replace("fp", "f"),
            "data": "synthetic (DESIGN.md §3; dynamic dictionary synth.make_src_ext)",
            "config": {"workload": args.workload, "task": "copy", "batch": B, "beam": K, "max_len": ML},
            "e2e": {"value": round(v, 1), "unit": "target tok/s", "h2d_bytes_per_step": int(2 * ids.nbytes + lens.nbytes),
                    "d2h_bytes_per_step": int(B * (ML * 8 + 12))},
            "same_workload_plain_model": {"value": round(vp, 1), "note": "onmt_translate of the model without the copy gate"},
            "copied_source_only_tokens": int((r["hyps"] >= cfg.v_tgt).sum())}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=list(synth.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-sentences", type=int, default=30)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-corpus", action="store_true")
    ap.add_argument("--corpus-sentences", type=int, default=0,
                    help="corpus-mode size (default: CORPUS[workload]; SURVEY §8(d) c4: 16384)")
    ap.add_argument("--vocab-parallel", action="store_true",
                    help="split the generator's vocabulary over the ranks (SURVEY §8(f) rank 4)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: a full batch per GPU (c2, c4); strong: the workload's batch sharded (c3, c5)")
    ap.add_argument("--task", default="translate", choices=["translate", "score", "translate_ex", "copy"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.task == "score":
        run_score(args)
    elif args.task == "translate_ex":
        run_translate_ex(args)
    elif args.task == "copy":
        run_copy(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
