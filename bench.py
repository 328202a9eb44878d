"""Benchmark: the VERSE/NCE training pass on the C2 workload.

Workload (BASELINE.json configs[1], SURVEY.md 8(d) "C2"): single-level
embedding-kernel microbench on a synthetic R-MAT graph, scale 20 (1,048,576
ids, all kept), 16,777,216 sampled edges, d=128, 3 negatives,
init_embedding(V, 128, seed=1), lr 0.035 constant.  One step = one vertex
pass over every non-isolated source = one launch of the training kernel.

Metric: sample-updates/s (TrainStats definition, trainer.py:238-240: passes x
non-isolated x (1+n_s)), with the kernel's achieved HBM GB/s against the
measured copy bandwidth (algorithmic bytes 8d(2+n_s)+12 per source).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun, one rank per GPU): each rank trains its own replica of the
workload (weak scaling, no data-path collective -- the in-memory pass does
not shard).  `--impl reference` times the reference's CPU path
(the oracle's C restatement of _train_pass, all host threads) on the same
workload; rank 0 only.
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

SCALE, SAMPLES, DIM, NNEG, SEED, LR = 20, 1 << 24, 128, 3, 7, 0.035
METRIC = "sample-updates/sec"
UNIT = "updates/s"


def workload_config():
    """The workload keys only -- both arms print exactly this dict (the
    driver compares them); run details go under "details"."""
    return {"workload": "C2 single-level VERSE pass: R-MAT scale 20 (2^20 ids, 2^24 sampled "
                        "edges, Graph500 a,b,c=0.57,0.19,0.19), d=128, n_neg=3",
            "scale": SCALE, "sampled_edges": SAMPLES, "dim": DIM, "negatives": NNEG,
            "rmat_seed": SEED, "lr": LR, "step": "one vertex pass (1 kernel launch)",
            "l2": "inputs larger than L2 (embedding matrix 512 MiB > 126 MB L2), no flush"}


def bytes_per_source(dim=DIM, n_neg=NNEG):
    return 8 * dim * (2 + n_neg) + 12


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "train_kernel_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clock/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _max_over_ranks(t):
    """all_reduce MAX (gloo takes host tensors: staged)."""
    import torch
    if torch.distributed.get_backend() == "gloo" and t.is_cuda:
        h = t.cpu()
        torch.distributed.all_reduce(h, op=torch.distributed.ReduceOp.MAX)
        return h.to(t.device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t


def dist_init():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # GB_DIST_BACKEND=gloo: a functional check of the multi-rank path on a
        # box with fewer GPUs than ranks (ranks share devices round-robin);
        # timing such a run means nothing
        backend = os.environ.get("GB_DIST_BACKEND", "nccl")
        dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def cpu_baseline(xadj, adj, seconds=12.0, warm=1):
    """Oracle C restatement of _train_pass (Hogwild, all host threads) on the
    same graph: bounded sample of whole passes."""
    from oracle import oracle as orc
    threads = orc.max_threads()
    V = len(xadj) - 1
    M = orc.init_embedding(V, DIM, 1)
    non_iso = int((np.diff(xadj) > 0).sum())
    for p in range(warm):
        orc.train_pass(xadj, adj, M, LR, NNEG, 1, 0, p, nthreads=threads)
    passes, t0 = 0, time.perf_counter()
    while True:
        orc.train_pass(xadj, adj, M, LR, NNEG, 1, 0, warm + passes, nthreads=threads)
        passes += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    upd = passes * non_iso * (1 + NNEG)
    return {"value": upd / el, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{passes} full C2 passes ({upd} updates) of oracle/gosh_oracle.c "
                      f"or_train_pass, {threads} threads, {el:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc
    xadj, adj = orc.rmat_graph(SCALE, SAMPLES, SEED)
    threads = orc.max_threads()
    V = len(xadj) - 1
    M = orc.init_embedding(V, DIM, 1)
    non_iso = int((np.diff(xadj) > 0).sum())
    for p in range(args.warmup):
        orc.train_pass(xadj, adj, M, LR, NNEG, 1, 0, p, nthreads=threads)
    t0 = time.perf_counter()
    for k in range(args.steps):
        orc.train_pass(xadj, adj, M, LR, NNEG, 1, 0, args.warmup + k, nthreads=threads)
    el = time.perf_counter() - t0
    value = args.steps * non_iso * (1 + NNEG) / el
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el * 1000.0 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 rows / f64 dot / f64 sigmoid",
        "data": "synthetic R-MAT (CPU generator, bit-identical to the GPU one)",
        "config": workload_config(),
        "details": {"parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} timed full C2 passes after {args.warmup} "
                                   f"warm-up passes, oracle/gosh_oracle.c or_train_pass"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours(args):
    import torch
    rank, world, local = dist_init()
    import paper_2008_12336_b200 as gb
    from paper_2008_12336_b200 import _lib
    dev = torch.device("cuda", local)

    t_build = time.perf_counter()
    G = gb.rmat_graph(SCALE, SAMPLES, SEED)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build
    xadj, adj = G.device_csr()
    V = G.num_vertices
    sources, non_iso = G.active_sources()
    M = torch.from_numpy(gb.init_embedding(V, DIM, 1)).to(dev)
    lrs = torch.tensor([np.float32(LR)], dtype=torch.float32, device=dev)
    status = _lib.new_status()
    stream = torch.cuda.current_stream()
    cap = gb.trainer.inflight_cap(gb.TrainConfig(dim=DIM), V)
    # the default path's flags (trainer._train_flags): vector-reduction
    # write-back, the reference's fp64 sigmoid
    flags = _lib.GB_TRAIN_ATOMIC if (not args.store_rows) else 0

    def launch(p):
        _lib.call("gb_train_passes", V, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(sources),
                  non_iso, _lib.ptr(M), DIM, NNEG,
                  1, 0, p, 1, 1 << 40, _lib.ptr(lrs), flags, cap,
                  _lib.ptr(status),
                  stream.cuda_stream)

    for p in range(args.warmup):
        launch(p)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            starts[k].record(stream)
            launch(args.warmup + k)
            ends[k].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    kern_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        t = _max_over_ranks(t)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    upd_per_step = non_iso * (1 + NNEG)
    value = world * upd_per_step / (ms_per_step / 1000.0)
    if int(status[0].item()):
        raise FloatingPointError("non-finite embedding during the benchmark")

    # e2e through the public API with host buffers: one train_level call per
    # step (one edge-scaled epoch = ceil(E/V) passes) on a host Graph (its CSR
    # is uploaded and its source list built inside the step), M copied in
    # from pinned host memory and back every step.
    M_host = torch.from_numpy(gb.init_embedding(V, DIM, 1)).pin_memory()
    cfg = gb.TrainConfig(dim=DIM, negative_samples=NNEG, seed=1, learning_rate=LR,
                         epoch_unit="edge-scaled", atomic_rows=(not args.store_rows))
    e2e_steps = max(2, min(args.steps // 10, 5))
    xh = torch.from_numpy(G.xadj).pin_memory().numpy()
    ah = torch.from_numpy(np.ascontiguousarray(G.adj)).pin_memory().numpy()
    csr_bytes = int(xh.nbytes + ah.nbytes)

    def host_graph():
        return gb.Graph(V, G.num_edges, xadj=xh, adj=ah)

    gb.train_level(host_graph(), M_host, cfg, 1)  # warm-up
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    te = time.perf_counter()
    e2e_upd = 0
    for _ in range(e2e_steps):
        st = gb.train_level(host_graph(), M_host, cfg, 1)
        e2e_upd += st.updates
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - te
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        t = _max_over_ranks(t)
        e2e_s = float(t.item())
    e2e_value = world * e2e_upd / e2e_s
    ppe = gb.trainer.passes_per_epoch(G, cfg)

    # the same pass with the fp32 cancellation-free sigmoid
    # (TrainConfig(fast_sigmoid=True)) instead of the reference's fp64 one:
    # same fp64 dot and write-back
    flags64 = _lib.GB_TRAIN_FAST_SIGMOID | (_lib.GB_TRAIN_ATOMIC if (not args.store_rows) else 0)

    def launch64(p):
        _lib.call("gb_train_passes", V, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(sources),
                  non_iso, _lib.ptr(M), DIM, NNEG, 1, 0, p, 1, 1 << 40, _lib.ptr(lrs), flags64,
                  cap, _lib.ptr(status), stream.cuda_stream)

    for p in range(3):
        launch64(10_000 + p)
    s64, e64 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n64 = max(3, args.steps // 2)
    torch.cuda.synchronize()
    s64.record(stream)
    for p in range(n64):
        launch64(20_000 + p)
    e64.record(stream)
    torch.cuda.synchronize()
    ms64 = s64.elapsed_time(e64) / n64

    bps = bytes_per_source()
    achieved = non_iso * bps / (kern_ms / 1000.0) / 1e9
    peak, peak_src = measured_peak()
    traffic = ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 rows / f64 dot / f64 sigmoid",
        "data": "synthetic R-MAT generated on device (seeded, Graph500 parameters)",
        "config": workload_config(),
        "details": {"vertices": V, "non_isolated_sources": non_iso, "arcs": G.num_edges,
                    "parallelism": "replicas" if world > 1 else "single GPU",
                    "inflight_groups_cap": cap, "graph_build_s": round(build_s, 3),
                    "kernel_flags": "default path: fp64 dot, fp64 sigmoid (the reference's), "
                                    "vector-reduction "
                                    "write-back of sample rows and source-row increments",
                    "row_writeback": "vector reductions" if (not args.store_rows) else "stores"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": non_iso * bps,
                     "bytes_per_source": bps, "kernel_ms": kern_ms, "peak_source": peak_src,
                     # real DRAM bytes (ncu, per launch) over the live kernel time: hub rows
                     # hit in L2, so this is below the algorithmic fraction
                     "dram_frac": (traffic / (kern_ms / 1000.0) / 1e9 / peak
                                   if traffic else None)},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": V * DIM * 4 + csr_bytes, "d2h_bytes_per_step": V * DIM * 4,
                "step": f"train_level(host Graph, M_pinned_host, edge-scaled, e_i=1): CSR "
                        f"upload + source list, {ppe} passes, M in/out", "steps": e2e_steps},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
        "fp32_sigmoid": {"value": upd_per_step / (ms64 / 1000.0), "unit": UNIT,
                         "kernel_ms": ms64, "frac": non_iso * bps / (ms64 / 1000.0) / 1e9 / peak,
                         "note": "same pass with the fp32 cancellation-free sigmoid "
                                 "(fast_sigmoid=True) instead of the reference's fp64 "
                                 "sigmoid/divide of the headline"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(xadj.cpu().numpy(), adj[: G.num_edges].cpu().numpy(),
                                            seconds=args.cpu_seconds)
    del M, xadj, adj, sources
    G = None
    torch.cuda.empty_cache()
    if world == 1 and not args.no_multilevel:
        line["multilevel_c3"] = multilevel_c3(args, cpu=not args.no_cpu_baseline)
        torch.cuda.empty_cache()
        anchor, _ = sharded_c3(args, 0, 1)
        anchor["config"] = sharded_config()
        anchor["note"] = ("N=1 point of the --gpus N strong-scaling line (K=2 parts, no "
                          "exchange); --gpus N>1 prints this workload as its headline")
        line["sharded_c3"] = anchor
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


C3_SCALE, C3_SAMPLES, C3_SEED, C3_DIM = 22, 126_000_000, 7, 128


def multilevel_c3(args, cpu=True):
    """The metric's second half, "embed wall time at equal AUCROC", on C3
    (BASELINE.json configs[2]: com-orkut-shaped R-MAT, 1 GPU): the public
    train_multilevel(host Graph) -> numpy matrix with the CLI defaults
    (cli.py:59-78: d=128, 1000 epochs, smoothing 0.3, lr 0.035, 3 negatives,
    vertex-pass), timed end to end -- CSR upload, coarsening, every level's
    training, expands, the matrix download -- on the train graph of the
    link-prediction split, then AUCROC of that embedding (device evaluator,
    1M+1M pair subsample).  The CPU leg is the oracle's restatement of the
    same embed on this box's host cores: the sequential coarsen_all (the
    reference's parity path) timed whole, each level's training timed on a
    bounded number of passes and extrapolated."""
    import torch
    import paper_2008_12336_b200 as gb
    from paper_2008_12336_b200.evaluate import LinkPredictionSetup
    t0 = time.perf_counter()
    g = gb.rmat_graph(C3_SCALE, C3_SAMPLES, C3_SEED, densify_ids=True)
    setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
    tg = setup.train_graph
    xh, ah = tg.xadj, tg.adj
    del g
    setup_s = time.perf_counter() - t0
    cfg = gb.TrainConfig(dim=C3_DIM, total_epochs=1000, smoothing_ratio=0.3, learning_rate=0.035,
                         negative_samples=3, seed=1, epoch_unit="vertex-pass")
    h = setup.hierarchy
    plan = gb.epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, h.depth).per_level
    updates = 0
    for i, gi in enumerate(h.graphs):
        ppe = gb.trainer.passes_per_epoch(gi, cfg)
        updates += int(plan[i]) * ppe * int((gi.degrees() > 0).sum()) * (1 + cfg.negative_samples)
    runs, M = [], None
    for _ in range(1 + args.c3_repeats):  # the first run is the warm-up
        fresh = gb.Graph(tg.num_vertices, tg.num_edges, xadj=xh, adj=ah)  # host arrays only
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        M = gb.train_multilevel(fresh, cfg)
        runs.append(time.perf_counter() - t1)
        del fresh
    embed_s = statistics.median(runs[1:])
    auc = setup.score(M)
    out = {"workload": "C3: R-MAT scale 22, 126M sampled edges, ids densified; link-prediction "
                       "train graph (test fraction 0.2, eval seed 1)",
           "vertices": tg.num_vertices, "arcs": tg.num_edges,
           "levels": [x.num_vertices for x in h.graphs],
           "config": "CLI defaults: d=128, 1000 epochs, smoothing 0.3, lr 0.035, n_neg 3, "
                     "vertex-pass, seed 1",
           "embed_s": embed_s, "embed_s_runs": runs[1:], "updates": updates,
           "updates_per_s": updates / embed_s,
           "h2d_bytes": int(xh.nbytes + ah.nbytes), "d2h_bytes": int(M.nbytes),
           "aucroc": auc, "aucroc_eval": "device evaluator, 1M train + 1M test positive pairs "
                                         "(+ as many negatives), LogRegConfig defaults",
           "setup_s": setup_s}
    if cpu:
        out["cpu_baseline"] = multilevel_cpu(xh, ah, cfg, plan, seconds=args.c3_cpu_seconds)
        out["cpu_baseline"]["speedup"] = out["cpu_baseline"]["embed_s_est"] / embed_s
    return out


def multilevel_cpu(xh, ah, cfg, plan, seconds=20.0):
    from oracle import oracle as orc
    threads = orc.max_threads()
    t0 = time.perf_counter()
    graphs, maps, _ = orc.coarsen_all(xh, ah, 100)
    coarsen_s = time.perf_counter() - t0
    per_level = max(seconds / len(graphs), 0.5)
    train_s = 0.0
    Mc = orc.init_embedding(len(graphs[-1][0]) - 1, cfg.dim, cfg.seed)
    timed = 0
    for i in range(len(graphs) - 1, -1, -1):
        x, a = graphs[i]
        V, E = len(x) - 1, int(x[-1])
        passes = int(plan[i]) * orc.passes_per_epoch(V, E, cfg.epoch_unit)
        n_run, t1 = 0, time.perf_counter()
        while n_run < passes:
            orc.train_pass(x, a, Mc, cfg.learning_rate, cfg.negative_samples, cfg.seed, i, n_run,
                           nthreads=threads)
            n_run += 1
            if time.perf_counter() - t1 >= per_level:
                break
        el = time.perf_counter() - t1
        train_s += el * passes / n_run
        timed += n_run
        if i > 0:
            Mc = orc.expand(Mc, maps[i - 1][0])
    return {"embed_s_est": coarsen_s + train_s, "coarsen_s": coarsen_s, "train_s_est": train_s,
            "cores": threads, "kind": "port",
            "sample": f"oracle/gosh_oracle.c: sequential coarsen_all timed whole; {timed} "
                      f"passes timed over the {len(graphs)} levels ({threads} threads), "
                      f"extrapolated to the plan's passes"}


SH_PASSES, SH_B = 80, 5


def sharded_config():
    """Workload keys of the multi-GPU line (identical for both arms)."""
    return {"workload": "C3 finest level trained by the part-pair tournament sharded over the "
                        "GPUs (SURVEY 8(e)): R-MAT scale 22, 126M sampled edges, ids densified, "
                        "d=128, n_neg=3, B=5, balanced pools; one step = an 80-vertex-pass "
                        "budget (rotations = 80 / (B K), K = 2 x GPUs parts); strong scaling",
            "scale": C3_SCALE, "sampled_edges": C3_SAMPLES, "rmat_seed": C3_SEED,
            "dim": C3_DIM, "negatives": NNEG, "batch": SH_B, "passes_per_step": SH_PASSES,
            "lr": LR, "l2": "inputs larger than L2 (1.3 GiB matrix), no flush"}


def sharded_cfg():
    import paper_2008_12336_b200 as gb
    return gb.TrainConfig(dim=C3_DIM, negative_samples=NNEG, seed=1, learning_rate=LR,
                          balanced_pools=True, epoch_unit="vertex-pass")


def sharded_c3(args, rank, world, print_line=True):
    """The tournament step on C3 over `world` ranks (one per GPU; world 1 =
    K=2 parts on one GPU, the strong-scaling anchor).  Each rank holds only
    its two parts (PartStore); every off-diagonal round ends with an NCCL
    P2P shift whose exposed time is measured with CUDA events."""
    import torch
    import paper_2008_12336_b200 as gb
    from paper_2008_12336_b200 import tournament as tn
    dev = torch.device("cuda", torch.cuda.current_device())
    g = gb.rmat_graph(C3_SCALE, C3_SAMPLES, C3_SEED, densify_ids=True)
    V = g.num_vertices
    cfg = sharded_cfg()
    local = [rank] if world > 1 else [0]
    store = tn.PartStore(V, C3_DIM, world, local, dev)
    store.init_random(cfg.seed)

    def step(ev=None):
        return tn.train_tournament_parts(g, store, cfg, SH_PASSES, batch_size=SH_B,
                                         exchange_events=ev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    events = []
    upd = sent = 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record(stream)
        launches = 0
        for _ in range(args.steps):
            st = step(events)
            upd += st["pos_updates"] + st["neg_updates"]
            sent += st["exchange_bytes"]
            launches += st["kernel_launches"]
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    total_ms = t0.elapsed_time(t1)
    exch_ms = sum(a.elapsed_time(b) for a, b in events)
    if world > 1:
        t = torch.tensor([total_ms, exch_ms], device=dev)
        t = _max_over_ranks(t)
        total_ms, exch_ms = (float(x) for x in t.tolist())
    value = upd / (total_ms / 1000.0)  # updates are summed over ranks by the driver
    bpu = 8 * C3_DIM + (8 * C3_DIM) / (SH_B * (1 + NNEG))
    peak, peak_src = measured_peak()
    out = {"value": value, "unit": UNIT, "ms_per_step": total_ms / args.steps, "K": 2 * world,
           "rotations_per_step": st["rotations"], "updates_per_step": upd // args.steps,
           "roofline": {"bound": "hbm", "achieved": value * bpu / 1e9 / world, "peak": peak,
                        "unit": "GB/s", "frac": value * bpu / 1e9 / world / peak,
                        "traffic": None, "bytes_per_update": bpu, "peak_source": peak_src,
                        "note": "per GPU, whole-step average including the exchanges"},
           "exchange": {"bytes_per_step": sent // args.steps,
                        "exposed_ms_per_step": exch_ms / args.steps,
                        "exposed_share": exch_ms / total_ms if total_ms else 0.0,
                        "nvlink_gbs_if_exposed": (sent / world / (exch_ms / 1000.0) / 1e9
                                                  if exch_ms > 0 and sent else None)},
           "part_bytes_per_gpu": store.device_bytes, "matrix_bytes": V * C3_DIM * 4,
           "gpu_launches": launches, "clocks": clk.summary()}
    del store
    return out, g


def run_sharded(args):
    """--gpus N > 1 (and --workload c3shard): the sharded C3 tournament step,
    strong scaling (the same total updates per step at every N)."""
    import torch
    rank, world, local = dist_init()
    import paper_2008_12336_b200 as gb
    from paper_2008_12336_b200 import tournament as tn
    res, g = sharded_c3(args, rank, world)
    # e2e through the public API: train_tournament(g, pinned host matrix) --
    # parts scattered from host memory, trained, gathered back every step
    cfg = sharded_cfg()
    M_host = torch.from_numpy(gb.init_embedding(g.num_vertices, C3_DIM, 1)).pin_memory()
    tn.train_tournament(g, M_host, cfg, SH_PASSES, batch_size=SH_B)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e2e_steps = max(2, min(args.steps, 3))
    te = time.perf_counter()
    e_upd = 0
    for _ in range(e2e_steps):
        st = tn.train_tournament(g, M_host, cfg, SH_PASSES, batch_size=SH_B)
        e_upd += st["pos_updates"] + st["neg_updates"]
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - te
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        t = _max_over_ranks(t)
        e2e_s = float(t.item())
    K = 2 * world
    part_bytes = -(-g.num_vertices // K) * C3_DIM * 4
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 rows / f64 dot / f64 sigmoid",
        "data": "synthetic R-MAT generated on device (seeded, Graph500 parameters)",
        "config": sharded_config(),
        "details": {"K": K, "vertices": g.num_vertices, "arcs": g.num_edges,
                    "rotations_per_step": res["rotations_per_step"],
                    "updates_per_step": res["updates_per_step"],
                    "parallelism": f"tournament over {world} GPU(s), one process each, "
                                   f"NCCL P2P part exchange",
                    "part_bytes_per_gpu": res["part_bytes_per_gpu"],
                    "matrix_bytes": res["matrix_bytes"]},
        "roofline": res["roofline"], "exchange": res["exchange"],
        "e2e": {"value": e_upd / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 2 * part_bytes,
                "d2h_bytes_per_step": g.num_vertices * C3_DIM * 4,
                "step": "train_tournament(g, M pinned host): 2 parts in, trained, all_gather "
                        "back to every rank's host matrix", "steps": e2e_steps},
        "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded_reference(args):
    """Reference arm of the multi-GPU line: the reference's partitioned pair
    step (oracle restatement of _fill_pool_side + _train_pool_side,
    bigtrain.py:164-238) on the same C3 graph and part count, all host
    threads, a bounded sample of pairs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle as orc
    threads = orc.max_threads()
    x, a = orc.rmat_graph(C3_SCALE, C3_SAMPLES, C3_SEED, densify_ids=True)
    V = len(x) - 1
    K = 2 * world
    bnd = (np.arange(K + 1, dtype=np.int64) * V) // K
    M = orc.init_embedding(V, C3_DIM, 1)
    upd, el, pairs = 0, 0.0, 0
    for k in range(args.warmup + args.steps):
        pa, pb = (k % K, (k + 1) % K)
        la, ha, lb, hb = int(bnd[pa]), int(bnd[pa + 1]), int(bnd[pb]), int(bnd[pb + 1])
        A = np.ascontiguousarray(M[la:ha])
        Bm = np.ascontiguousarray(M[lb:hb])
        t0 = time.perf_counter()
        tj = orc.fill_pool_side(x, a, la, ha, lb, hb, SH_B, 7 + k, 0)
        pos = orc.train_pool_side(A, Bm, tj, lb, hb - lb, NNEG, LR, 7 + k, 2, nthreads=threads)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            upd += pos * (1 + NNEG)
            el += dt
            pairs += 1
    value = upd / el
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1000.0 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 rows / f64 dot / f64 sigmoid", "data": "synthetic R-MAT (CPU generator, bit-identical "
                                              "to the GPU one)",
        "config": sharded_config(),
        "details": {"parallelism": f"{threads} host threads", "K": K},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{pairs} pair sides (fill_pool_side + train_pool_side, "
                                   f"K={K} parts of the C3 graph), oracle/gosh_oracle.c"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def run_tournament(args):
    """Part-pair tournament (tournament.py) on the C2 graph: K = 2N parts,
    one step = --rotations rotations (every pair once per rotation, K(K+1)/2
    pair launches, parts exchanged over NCCL between rounds).  Units: positive +
    negative updates, B=5 positives per source per pair side."""
    import torch
    rank, world, local = dist_init()
    import paper_2008_12336_b200 as gb
    from paper_2008_12336_b200 import tournament as tn
    dev = torch.device("cuda", local)
    B = 5
    dim = args.dim or DIM
    G = gb.rmat_graph(SCALE, SAMPLES, SEED)
    V = G.num_vertices
    cfg = gb.TrainConfig(dim=dim, negative_samples=NNEG, seed=1, learning_rate=LR,
                         atomic_rows=(not args.store_rows))
    M = torch.from_numpy(gb.init_embedding(V, dim, 1)).to(dev)

    vr = max(1, args.virtual_ranks)
    K = 2 * world if world > 1 else 2 * vr
    R = max(1, args.rotations)

    def step():
        # an R * B * K vertex-pass budget = R rotations (tournament_rotations)
        return tn.train_tournament(G, M, cfg, R * B * K, batch_size=B, gather=False,
                                   num_ranks=None if world > 1 else vr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record(stream)
        upd = launches = 0
        for _ in range(args.steps):
            st = step()
            upd += st["pos_updates"] + st["neg_updates"]
            launches += st["kernel_launches"]
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    total_ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        t = _max_over_ranks(t)
        total_ms = float(t.item())
    value = upd / (total_ms / 1000.0)  # pos_updates are already summed over ranks
    bpu = 8 * dim + (8 * dim) / (B * (1 + NNEG))
    peak, peak_src = measured_peak()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 rows / f64 dot / f64 sigmoid",
        "data": "synthetic R-MAT generated on device (seeded, Graph500 parameters)",
        "config": ({
            "workload": f"part-pair tournament on the C2 graph, K={K} parts, B={B}, d={dim}",
            "dim": dim,
            "step": f"{R} rotations: each K(K+1)/2 pairs, K-1 part exchanges "
                    "(one process: rotation 0 eager, the rest replayed from a CUDA graph)",
            "rotation_graph": os.environ.get("GB_ROTATION_GRAPH", "auto"),
            "parallelism": f"tournament over {world} GPU(s)"
                           + (f" ({vr} virtual ranks)" if world == 1 and vr > 1 else ""),
            "vertices": V, "pool_mode": os.environ.get("GB_POOL_MODE", "compact")}),
        "roofline": {"bound": "hbm", "achieved": value * bpu / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": value * bpu / 1e9 / world / peak, "traffic": None,
                     "bytes_per_update": bpu, "peak_source": peak_src,
                     "note": "whole-step average incl. exchanges, per GPU"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-multilevel", action="store_true",
                    help="skip the C3 multilevel embed + AUCROC field")
    ap.add_argument("--c3-repeats", type=int, default=3)
    ap.add_argument("--c3-cpu-seconds", type=float, default=20.0)
    ap.add_argument("--workload", choices=["auto", "c2", "c3shard", "tournament"],
                    default="auto",
                    help="auto: c2 at N=1 (BASELINE configs[1]), c3shard at N>1 (configs[2] "
                         "strong scaling)")
    ap.add_argument("--dim", type=int, default=0,
                    help="tournament workload: embedding dimension (default 128; C5 uses 256)")
    ap.add_argument("--rotations", type=int, default=32,
                    help="tournament workload: rotations per step")
    ap.add_argument("--virtual-ranks", type=int, default=1,
                    help="tournament on one GPU: run the schedule of R ranks (K = 2R parts) "
                         "in this process")
    ap.add_argument("--store-rows", action="store_true",
                    help="write sample rows back with plain stores instead of the default "
                         "vector reductions (GB_TRAIN_ATOMIC off)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    workload = args.workload
    if workload == "auto":
        workload = "c3shard" if max(world, args.gpus) > 1 else "c2"
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator size in the log
    if args.impl == "reference":
        if workload == "c3shard":
            run_sharded_reference(args)
        else:
            run_reference(args)
    elif workload == "tournament":
        run_tournament(args)
    elif workload == "c3shard":
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
