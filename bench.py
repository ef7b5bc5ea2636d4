#!/usr/bin/env python
"""Benchmark of the hot path: one step = a1..a9 over one
profiling table — ingest (label + value tables + bins), level-wise CART to
depth D, and batched selection of the same table's feature vectors.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU); the table's rows are split
into contiguous shards (strong scaling: the C4 table is 1e8 rows in total) and
the per-level histograms are summed with NCCL inside libadapt.so.  Rank 0
prints ONE JSON line.  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import signal
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "CART train samples/s and variant selections/s at 1/2/4/8 B200; % HBM peak"
WORKLOADS = {
    "C4": "C4: 1e8-row profiling table, 16 features, 48 variants (offload x threads x block), "
          "depth-12 CART + selection of the same 1e8 vectors",
    "C3": "C3: 1e6-row table, 8 features, 6 variants (GPU block size), depth-12 CART + selection",
    "C2": "C2 region 0: 3.3e4-row table, 4 features, 7 variants (num_threads), depth 8",
    "C1": "C1: 512 profiled samples, 1 feature (trip count), host vs GPU offload, depth 4",
}
KERNEL_PHASES = ("discover", "ingest", "values", "merge", "zero", "partition", "tag", "hist", "subtract", "split", "winner", "bootstrap",
                 "decide", "select")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, from the latest
    committed ncu --set full captures (profiles/roundNN/ncu_traffic.json)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "round*", "ncu_traffic.json")))
    if not files:
        return {}
    with open(files[-1]) as fh:
        return json.load(fh)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
                start_new_session=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.25)
            os.killpg(self.proc.pid, signal.SIGTERM)
            self.out, _ = self.proc.communicate()

    def summary(self):
        if not getattr(self, "out", ""):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count(), model


def cpu_baseline(cfg, rows: int, depth: int, omp: bool = False):
    """The oracle as it stands (plain C), on a bounded sample of the same
    workload: the first `rows` rows of the table, labels + tree + select.
    omp=True: the same source built with -fopenmp (liboracle_omp.so: features
    of a node and vectors in parallel, identical results) on all host cores."""
    import oracle

    X, T = synth.generate(cfg, 0, rows)
    t0 = time.perf_counter()
    y = oracle.labels(T)
    tree = oracle.train(X, y, cfg.V, depth, omp=omp)
    oracle.select(tree, X, omp=omp)
    dt = time.perf_counter() - t0
    return rows / dt, dt


def bench_c5(args, ad, adist, torch, dev, stream, rank: int, world: int, peak: float):
    """batched selection of M = 1e9 C4-shaped feature vectors
    (seed 7, sharded over the ranks) by (i) a depth-16 tree trained by the
    engine on a 1e7-row C4-shaped table (seed 5) and (ii) the synthetic complete
    depth-16 tree (seed 6, the worst case).  Each timed launch is one
    adapt_select_batch over the rank's whole shard (64 GB at P=1: > L2)."""
    import dataclasses

    cfg = dataclasses.replace(synth.CONFIGS["C4"], D=16)
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev)
    Nt = args.c5_train_rows
    tlo, thi = adist.shard_bounds(Nt, rank, world)
    Xt = torch.empty((thi - tlo, cfg.F), dtype=torch.float32, device=dev)
    Tt = torch.empty((thi - tlo, cfg.V), dtype=torch.float32, device=dev)
    synth.generate_device(cfg, tlo, thi - tlo, Xt.data_ptr(), Tt.data_ptr(), g.data_ptr(), o.data_ptr(),
                          stream.cuda_stream, seed=5)
    trained = ad.adapt_region_create("bench_c5_trained", cfg.F, cfg.V, "dtree,depth=16", 0)
    ad.adapt_record_table(trained, Xt, Tt, thi - tlo, True, stream)
    ad.adapt_train(trained, stream)
    del Xt, Tt
    cols = synth.random_tree(cfg, 16, seed=6)
    tree = np.zeros(len(cols["feature"]), ad.NODE_DTYPE)
    for k, v in cols.items():
        tree[k] = v
    complete = ad.adapt_region_create("bench_c5_complete", cfg.F, cfg.V, "dtree,depth=16", 0)
    ad.adapt_set_tree(complete, tree)
    M = args.c5_vectors
    lo, hi = adist.shard_bounds(M, rank, world)
    m = hi - lo
    X = torch.empty((m, cfg.F), dtype=torch.float32, device=dev)
    out = torch.empty(m, dtype=torch.int32, device=dev)
    synth.generate_device(cfg, lo, m, X.data_ptr(), 0, g.data_ptr(), o.data_ptr(), stream.cuda_stream,
                          seed=7)
    res = {"workload": "C5: depth-16 trees evaluated on 1e9 C4-shaped feature vectors (16 f32 "
                       "features), sharded over the ranks",
           "vectors": M, "bytes_per_vector": 4 * cfg.F + 4, "steps": args.steps, "warmup": args.warmup,
           "l2": "X (%.0f GB per rank) exceeds the 126 MB L2; no flush needed" % (m * 4 * cfg.F / 1e9)}
    for name, h in (("trained", trained), ("complete", complete)):
        for _ in range(max(args.warmup, 1)):
            ad.adapt_select_batch(h, X, m, out, stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ad.adapt_select_batch(h, X, m, out, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = adist.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
        gbs = m * (4 * cfg.F + 4) / (ms / 1e3) / 1e9  # rank-local bytes / max-over-ranks time
        res[name] = {"tree_nodes": int(len(ad.adapt_get_tree(h))), "ms_per_batch": ms,
                     "selections_per_s": M / (ms / 1e3),
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                                  "frac": gbs / peak}}
    ad.adapt_region_destroy(trained)
    ad.adapt_region_destroy(complete)
    del X, out
    torch.cuda.empty_cache()
    return res


def bench_kfold(args, ad, adist, torch, dev, stream, rank: int, world: int):
    """The paper's evaluation protocol as a GPU workload: K = 4 groups,
    10 shuffles, m = 1/2/3 training groups (Adaptive-25/50/75) = 120 depth-D
    models on the C3 table (1e6 rows, sharded), each tested on its held-out rows."""
    cfg = synth.CONFIGS["C3"]
    N = cfg.N
    lo, hi = adist.shard_bounds(N, rank, world)
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev)
    X = torch.empty((hi - lo, cfg.F), dtype=torch.float32, device=dev)
    T = torch.empty((hi - lo, cfg.V), dtype=torch.float32, device=dev)
    synth.generate_device(cfg, lo, hi - lo, X.data_ptr(), T.data_ptr(), g.data_ptr(), o.data_ptr(),
                          stream.cuda_stream)
    h = ad.adapt_region_create("bench_kfold", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)

    def run():
        out = []
        for m in (1, 2, 3):
            ad.adapt_record_table(h, X, T, hi - lo, True, stream)
            out.append(ad.adapt_kfold(h, 4, m, 10, 1, stream))
        return out

    for _ in range(max(args.warmup, 1)):
        run()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = adist.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    ad.adapt_region_destroy(h)
    acc = {f"adaptive_{25 * m}": float(res[m - 1]["n_correct"].sum() / res[m - 1]["n_test"].sum())
           for m in (1, 2, 3)}
    slow = {f"adaptive_{25 * m}": float(res[m - 1]["t_selected"].sum() / res[m - 1]["t_best"].sum())
            for m in (1, 2, 3)}
    return {"workload": "C3 table (1e6 rows, 8 features, 6 variants), K=4 groups x 10 shuffles x "
                        "m=1/2/3 training groups = 120 depth-12 models, each tested on its held-out rows",
            "models": 120, "ms": ms, "models_per_s": 120 / (ms / 1e3),
            "model_rows_per_s": sum(int(r["n_train"].sum()) for r in res) / (ms / 1e3),
            "test_accuracy": acc, "time_selected_over_best": slow}


def bench_c2(args, ad, adist, torch, dev, stream, rank: int, world: int):
    """C2 as BASELINE.json states it: 3 regions (region = row mod 3, R15), 1e5
    profiled samples in total, 7 num_threads variants, depth 8 — the three
    region trees in one adapt_train_many (one multi-root frontier over the
    union table), timed against training the regions one by one."""
    cfg = synth.CONFIGS["C2"]
    X, T = synth.generate(cfg, 0, cfg.N)
    hs, keep = [], []
    for r in range(cfg.regions):
        rows = synth.region_rows(cfg, r)
        lo, hi = adist.shard_bounds(len(rows), rank, world)
        dX = torch.from_numpy(np.ascontiguousarray(X[rows[lo:hi]])).to(dev)
        dT = torch.from_numpy(np.ascontiguousarray(T[rows[lo:hi]])).to(dev)
        keep.append((dX, dT))
        hs.append(ad.adapt_region_create(f"bench_c2_r{r}", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0))

    def record():
        for h, (dX, dT) in zip(hs, keep):
            ad.adapt_record_table(h, dX, dT, dX.shape[0], True, stream)

    def fused():
        record()
        ad.adapt_train_many(hs, stream)

    def one_by_one():
        record()
        for h in hs:
            ad.adapt_train(h, stream)

    res = {"workload": "C2: 3 regions (row mod 3), 1e5 samples in total, 4 features, 7 variants, depth 8",
           "regions": cfg.regions, "rows": cfg.N, "steps": args.steps}
    for name, fn in (("train_many_ms", fused), ("one_by_one_ms", one_by_one)):
        for _ in range(max(args.warmup, 1)):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        res[name] = adist.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    res["samples_per_s"] = cfg.N / (res["train_many_ms"] / 1e3)
    for h in hs:
        ad.adapt_region_destroy(h)
    return res


def bench_c1(args, ad, torch, dev, stream):
    """C1 at the paper's own scale (Table 4: 60-280 us to train a
    depth-2 tree on ~10 tuples, 7-20 ns per inference): latency of one
    adapt_train on C1's 512 profiled samples (depth 4, device tables; the call
    returns with the tree on the host) and of one host-side get_policy walk
    (adapt_select), host wall clock, median of many calls."""
    cfg = synth.CONFIGS["C1"]
    X, T = synth.generate(cfg, 0, cfg.N)
    dX, dT = torch.from_numpy(X).to(dev), torch.from_numpy(T).to(dev)
    h = ad.adapt_region_create("bench_c1", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)
    lat = []
    for i in range(60):
        ad.adapt_record_table(h, dX, dT, cfg.N, True, stream)
        t0 = time.perf_counter()
        ad.adapt_train(h, stream)
        if i >= 10:
            lat.append((time.perf_counter() - t0) * 1e6)
    xs = [X[i] for i in range(0, cfg.N, 7)]
    t0 = time.perf_counter()
    reps = 200
    for _ in range(reps):
        for x in xs:
            ad.adapt_select(h, x)
    sel_ns = (time.perf_counter() - t0) * 1e9 / (reps * len(xs))
    ad.adapt_region_destroy(h)
    c_ns = None
    exe = os.path.join(ROOT, "scripts", "select_latency")
    if os.path.exists(exe):  # the same walk timed from C: no Python in the loop
        import tempfile

        with tempfile.TemporaryDirectory() as td:
            xf, tf = os.path.join(td, "X.f32"), os.path.join(td, "T.f32")
            X.tofile(xf)
            T.tofile(tf)
            r = subprocess.run([exe, xf, tf, str(cfg.N), str(cfg.F), str(cfg.V), f"dtree,depth={cfg.D}",
                                "2000"], capture_output=True, text=True, timeout=120)
            if r.returncode == 0:
                c_ns = json.loads(r.stdout)["ns_per_call"]
    return {"workload": "C1: 512 profiled samples, 1 feature, 2 variants, depth 4",
            "train_us_median": statistics.median(lat), "train_us_min": min(lat),
            "select_host_ns_per_call": sel_ns,
            "select_host_ns_per_call_c": c_ns,
            "note": "select_host_ns_per_call: adapt_select through the ctypes binding (includes "
                    "Python call overhead); select_host_ns_per_call_c: the same C-ABI call timed in a "
                    "C loop (scripts/select_latency.c, 2000 passes over the 512 vectors); paper "
                    "Table 4: 60-280 us training, 7-20 ns per inference on the host"}


def bench_c3(args, ad, adist, torch, dev, stream, rank: int, world: int, peak: float):
    """C3 as BASELINE.json states it: 1e6 samples, 8 features, 6 block-size
    variants, depth 12, 256 bins — adapt_record_table + adapt_train per step."""
    cfg = synth.CONFIGS["C3"]
    lo, hi = adist.shard_bounds(cfg.N, rank, world)
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev)
    X = torch.empty((hi - lo, cfg.F), dtype=torch.float32, device=dev)
    T = torch.empty((hi - lo, cfg.V), dtype=torch.float32, device=dev)
    synth.generate_device(cfg, lo, hi - lo, X.data_ptr(), T.data_ptr(), g.data_ptr(), o.data_ptr(),
                          stream.cuda_stream)
    h = ad.adapt_region_create("bench_c3", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)

    def step():
        ad.adapt_record_table(h, X, T, hi - lo, True, stream)
        ad.adapt_train(h, stream)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = adist.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    levels = ad.adapt_train_stats(h)
    rows = sum((lv["rows_part"] if i else hi - lo) for i, lv in enumerate(levels) if lv["nodes"])
    byts = (4 * cfg.F + 4 * cfg.V + cfg.F + 1) * cfg.N + (cfg.F + 1) * rows * world
    ad.adapt_region_destroy(h)
    return {"workload": "C3: 1e6-row table, 8 features, 6 variants (GPU block size), depth 12",
            "ms": ms, "train_samples_per_s": cfg.N / (ms / 1e3),
            "survey_bytes": byts, "hbm_frac": byts / (ms / 1e3) / 1e9 / peak,
            "note": "latency/launch-bound at this size (SURVEY 8(d): 26 us at 100% of HBM)"}


def bench_scaling_proxy(args, ad, torch, dev, stream, full_levels, full_ms: float, peak: float):
    """Multi-GPU readiness without an 8-GPU box: C4's per-rank work
    at P = 8 — the first 1.25e7 rows of the table — on this one GPU, timed like
    the main step, with (i) the share of the step in which no engine kernel runs
    (host bookkeeping and launch gaps), per level and in total, and (ii) the
    projected per-level exchange at P = 8: the default all-reduce moves
    2 (P-1)/P x the direct nodes' histogram bytes per rank (the same histogram
    sizes as the full table's, `full_levels`), timed at the measured 8-rank
    NVLink all-reduce bus bandwidth of 725 GB/s (B200_PROFILING.md)."""
    cfg = synth.CONFIGS["C4"]
    P = 8
    n = cfg.N // P
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev)
    X = torch.empty((n, cfg.F), dtype=torch.float32, device=dev)
    T = torch.empty((n, cfg.V), dtype=torch.float32, device=dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    synth.generate_device(cfg, 0, n, X.data_ptr(), T.data_ptr(), g.data_ptr(), o.data_ptr(),
                          stream.cuda_stream)
    h = ad.adapt_region_create("bench_proxy", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)

    def step():
        ad.adapt_record_table(h, X, T, n, True, stream)
        ad.adapt_train(h, stream)
        ad.adapt_select_batch(h, X, n, out, stream)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    ad.adapt_profile_reset()
    ad.adapt_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ad.adapt_profile_enable(False)
    prof = ad.adapt_profile_get()
    ms = e0.elapsed_time(e1) / args.steps
    kern_ms = sum(v["ms"] for k, v in prof.items() if k.split("_L")[0] in KERNEL_PHASES) / args.steps
    lv_ms = {}
    for k, v in prof.items():
        base, _, lv = k.partition("_L")
        if lv.isdigit() and base in KERNEL_PHASES:
            lv_ms[int(lv)] = lv_ms.get(int(lv), 0.0) + v["ms"] / args.steps
    levels = ad.adapt_train_stats(h)
    split_ms = {}
    for k, v in prof.items():
        base, _, lv = k.partition("_L")
        if base in ("split",) and lv.isdigit():
            split_ms[int(lv)] = v["ms"] / args.steps
    winner_ms = prof.get("winner", {"ms": 0.0})["ms"] / args.steps
    per_level = []
    for d, lv in enumerate(levels):
        full = full_levels[d] if d < len(full_levels) else lv
        # default exchange at P > 1 (engine.cpp hist_comm_rs): reduce-scatter of
        # every node's histogram by owner ((P-1)/P of the level's histogram
        # bytes per rank) + the winner all-gather (small)
        rsb = (P - 1) / P * full.get("hist_bytes", 0)
        per_level.append({"nodes": lv["nodes"], "kernel_ms": round(lv_ms.get(d, 0.0), 4),
                          "split_ms": round(split_ms.get(d, 0.0), 4),
                          "reduce_scatter_bytes_per_rank": int(rsb),
                          "reduce_scatter_ms_at_725GBps": round(rsb / 725e9 * 1e3, 4)})
    ad.adapt_region_destroy(h)
    del X, T, out
    torch.cuda.empty_cache()
    comm_ms = sum(x["reduce_scatter_ms_at_725GBps"] for x in per_level)
    owner_saving = (sum(split_ms.values()) + winner_ms) * (P - 1) / P  # owners search 1/P of the nodes
    step_p8 = ms - owner_saving + comm_ms
    return {"workload": "C4 rows [0, 1.25e7): one rank's shard at P = 8 (strong scaling of the 1e8 table)",
            "rows": n, "ms_per_step": ms, "kernel_ms_per_step": kern_ms,
            "host_idle_share": max(0.0, 1 - kern_ms / ms),
            "split_winner_ms_per_step": sum(split_ms.values()) + winner_ms,
            "projected_exchange_ms_per_step": comm_ms,
            "projected_step_ms_p8": step_p8,
            "projected_speedup_p8": full_ms / step_p8,
            "levels": per_level,
            "note": "projection for P = 8 with the default exchange (reduce-scatter by node "
                    "ownership): this shard's step, minus (P-1)/P of the split search and winner "
                    "kernels (each owner searches 1/P of the nodes), plus the per-level exchange "
                    "at 725 GB/s added serially (no overlap)"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    rows = args.ref_rows or {"C4": 300_000, "C3": 300_000}.get(args.config, cfg.N)
    oracle_import = __import__("oracle")
    oracle_import.build()
    times = []
    for i in range(args.warmup + args.steps):
        v, dt = cpu_baseline(cfg, rows, cfg.D)
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = rows / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "sample_rows": rows},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "oracle",
                         "sample": f"first {rows} rows of {args.config} (labels + depth-{cfg.D} "
                                   f"exact CART + select), single-threaded C oracle",
                         "host_cores": host_cpu()[0], "cpu_model": host_cpu()[1]},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=0, help="override table rows (testing only)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=0)
    ap.add_argument("--depth", type=int, default=0, help="override the config's depth (testing only)")
    ap.add_argument("--model", default="", help="model_type override, e.g. 'rfc,10,4' (P:257)")
    ap.add_argument("--records", type=int, default=20_000_000, help="record-path batch size")
    ap.add_argument("--no-records", action="store_true")
    ap.add_argument("--c5-vectors", type=int, default=1_000_000_000, help="C5 batch size (SURVEY §8(d))")
    ap.add_argument("--c5-train-rows", type=int, default=10_000_000)
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-kfold", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--no-proxy", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    os.environ.setdefault("ADAPT_PROFILE_LEVELS", "1")  # per-level phase names (SURVEY §8(d) reporting)
    import paper_2303_08873_b200 as ad
    from paper_2303_08873_b200 import dist as adist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    adist.init_nccl(local, rank, world)

    cfg = synth.CONFIGS[args.config]
    if args.depth:
        import dataclasses
        cfg = dataclasses.replace(cfg, D=args.depth)
    N = args.rows or (cfg.N if cfg.regions == 1 else len(synth.region_rows(cfg, 0)))
    lo, hi = adist.shard_bounds(N, rank, world)
    n = hi - lo
    stream = torch.cuda.current_stream()
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev)
    X = torch.empty((n, cfg.F), dtype=torch.float32, device=dev)
    T = torch.empty((n, cfg.V), dtype=torch.float32, device=dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    synth.generate_device(cfg, lo, n, X.data_ptr(), T.data_ptr(), g.data_ptr(), o.data_ptr(),
                          stream.cuda_stream)
    torch.cuda.synchronize()
    model = args.model or f"dtree,depth={cfg.D}"
    h = ad.adapt_region_create(f"bench_{args.config}", cfg.F, cfg.V, model, 0)

    def step():
        ad.adapt_record_table(h, X, T, n, True, stream)
        ad.adapt_train(h, stream)
        ad.adapt_select_batch(h, X, n, out, stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        step()
    barrier()
    # the timed region runs without the engine's per-phase events; the phase
    # breakdown (and the roofline's kernel time) comes from separate steps
    # with them on, right after
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = adist.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    ad.adapt_profile_reset()
    ad.adapt_profile_enable(True)
    prof_steps = max(1, min(args.steps, 5))
    for _ in range(prof_steps):
        step()
    barrier()
    ad.adapt_profile_enable(False)
    prof = ad.adapt_profile_get()
    tree = ad.adapt_get_tree(h)
    levels = ad.adapt_train_stats(h)

    # ---- end to end through the public API with HOST buffers ----
    e2e = None
    if not args.no_e2e:
        hX = torch.empty((n, cfg.F), dtype=torch.float32, pin_memory=True)
        hT = torch.empty((n, cfg.V), dtype=torch.float32, pin_memory=True)
        hout = torch.empty(n, dtype=torch.int32, pin_memory=True)
        hX.copy_(X)
        hT.copy_(T)
        he = ad.adapt_region_create(f"bench_e2e_{args.config}", cfg.F, cfg.V, model, 0)

        def step_host():  # the table crosses PCIe once: the select walks the library's copy
            ad.adapt_record_table(he, hX, hT, n, False, stream)
            ad.adapt_train(he, stream)
            ad.adapt_select_table(he, hout, stream)

        step_host()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            step_host()
        barrier()
        e2e_ms = adist.max_over_ranks((time.perf_counter() - t0) * 1e3 / args.e2e_steps, dev)
        assert np.array_equal(hout.numpy(), out.cpu().numpy()), "e2e selections differ from device path"
        e2e = {"value": N / (e2e_ms / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": int(N * (4 * cfg.F + 4 * cfg.V)),
               "d2h_bytes_per_step": int(N * 4), "ms_per_step": e2e_ms, "steps": args.e2e_steps,
               "timer": "host wall clock around synchronous C-ABI calls, max over ranks",
               "calls": "adapt_record_table (pinned host table) + adapt_train + adapt_select_table "
                        "(selections of the same vectors from the library's device copy, to host)"}
        del hX, hT, hout

    # ---- the GPU record path: long-format records -> wide rows ----
    rec = None
    if not args.no_records and world == 1:
        M = args.records
        g = torch.Generator(device=dev).manual_seed(5)
        rows = torch.randint(0, min(n, 500_000), (M,), device=dev, generator=g)
        rv = torch.randint(0, cfg.V, (M,), device=dev, generator=g, dtype=torch.int32)
        rX = X[rows].contiguous()
        rns = T[rows, rv.long()].to(torch.int64).contiguous()
        hr = ad.adapt_region_create(f"bench_rec_{args.config}", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)
        ad.adapt_record_batch(hr, rX, rv, rns, M, True, stream)
        ad.adapt_train(hr, stream)  # warm-up
        ad.adapt_profile_reset()
        ad.adapt_profile_enable(True)
        ad.adapt_train(hr, stream)
        ad.adapt_profile_enable(False)
        rp = ad.adapt_profile_get().get("records", {"ms": 0.0, "launches": 0, "bytes": 0.0})
        wide = ad.adapt_region_info(hr)["num_rows"]
        rec = {"records": M, "distinct_vectors": int(len(ad.adapt_get_wide_table(hr)[0])),
               "ms": rp["ms"], "records_per_s": M / (rp["ms"] / 1e3) if rp["ms"] else None,
               "launches": rp["launches"],
               "note": "device-batch records from the first 5e5 C4 rows x random variants; "
                       "GPU aggregation only (the train that follows is the main metric's path)"}
        del rX, rns, rv, rows
        _ = wide

    peak, peak_src = peaks()
    c5 = None
    if not args.no_c5 and args.config == "C4":
        ad.adapt_region_destroy(h)
        del X, T, out
        torch.cuda.empty_cache()
        c5 = bench_c5(args, ad, adist, torch, dev, stream, rank, world, peak)
    c1 = bench_c1(args, ad, torch, dev, stream) if (not args.no_c2 and args.config == "C4" and world == 1) else None
    c2 = None
    if not args.no_c2 and args.config == "C4":
        c2 = bench_c2(args, ad, adist, torch, dev, stream, rank, world)
    kfold = None
    if not args.no_kfold and args.config == "C4":
        kfold = bench_kfold(args, ad, adist, torch, dev, stream, rank, world)
    c3 = None
    if not args.no_c2 and args.config == "C4":
        c3 = bench_c3(args, ad, adist, torch, dev, stream, rank, world, peak)
    proxy = None
    if not args.no_proxy and args.config == "C4" and world == 1:
        proxy = bench_scaling_proxy(args, ad, torch, dev, stream, levels, ms, peak)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # per-level phases (partition_L03, hist_L03, split_L03) -> the levels table;
    # everything else is aggregated per kernel phase
    per_level = {}
    kern = {}
    for k, v in prof.items():
        base, _, lv = k.partition("_L")
        if base not in KERNEL_PHASES:
            continue
        if lv.isdigit():
            per_level.setdefault(int(lv), {})[base] = round(v["ms"] / prof_steps, 4)
        a = kern.setdefault(base, {"launches": 0, "ms": 0.0, "bytes": 0.0})
        a["launches"] += v["launches"]
        a["ms"] += v["ms"]
        a["bytes"] += v["bytes"]
    for i, lv in enumerate(levels):
        lv["ms"] = per_level.get(i, {})
    # SURVEY §8(d) algorithmic bytes (what the method must move, not what this
    # implementation moves): ingest 4F+4V read + F+1 written per row; training
    # (F+1) per row of an active node per level; selection 4F read + 4 written
    # per vector.  Per kernel phase: the phase's rows x that per-row figure.
    F, V = cfg.F, cfg.V
    rows_part = sum(lv["rows_part"] for lv in levels)
    rows_hist = sum(lv["rows_hist"] for lv in levels)
    alg = {"ingest": (4 * F + 4 * V + F + 1) * n * prof_steps,
           "partition": (F + 1) * rows_part * prof_steps,
           "hist": (F + 1) * rows_hist * prof_steps,
           "select": (4 * F + 4) * n * prof_steps}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    d = kern[dom]
    alg_dom = alg.get(dom)
    achieved = alg_dom / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 and alg_dom else None
    impl = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 and d["bytes"] > 0 else None
    step_ms_phases = {k: round(v["ms"] / prof_steps, 4) for k, v in kern.items()}
    traffic = ncu_traffic().get(dom.split("_L")[0])
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                "traffic_source": (f'{traffic["source"]} ({traffic["capture"]}, one ncu --set full '
                                   f'capture)') if traffic else None,
                "peak_source": peak_src,
                "alg_bytes_per_launch": (alg_dom or 0) / max(d["launches"], 1),
                "alg_bytes_rule": "SURVEY 8(d): ingest 4F+4V+F+1 per row; partition / hist (F+1) per row "
                                  "they process (a tagged level's histogram reads its parents' rows); "
                                  "select 4F+4 per vector",
                "ms_per_launch": d["ms"] / max(d["launches"], 1),
                "impl_bytes_per_launch": d["bytes"] / max(d["launches"], 1),
                "impl_frac": (impl / peak) if impl else None}
    # the whole level loop against SURVEY §8(d)'s level figure: (F+1) bytes per
    # row of an active node per level
    loop_ms = sum(step_ms_phases.get(k, 0) for k in ("partition", "tag", "hist", "zero", "subtract", "split",
                                                   "winner", "decide", "fused"))
    loop_rows = sum((lv["rows_part"] if i else n) for i, lv in enumerate(levels) if lv["nodes"])
    loop_bytes = (F + 1) * loop_rows * world
    two_level = (not os.environ.get("ADAPT_ONE_LEVEL") and os.environ.get("ADAPT_TWO_LEVEL") != "0" and world == 1
                 and (os.environ.get("ADAPT_TWO_LEVEL") == "1" or N >= 1 << 24))
    level_loop = {"schedule": ("two-level row moves: TAG + MOVE4, partition into the last level" if two_level
                               else "partition every level"),
                  "phases": "partition, tag, hist, zero, subtract, split, winner, decide",
                  "survey_bytes_per_step": loop_bytes, "ms_per_step": loop_ms,
                  "achieved_gbs": loop_bytes / (loop_ms / 1e3) / 1e9 if loop_ms else None,
                  "frac": loop_bytes / (loop_ms / 1e3) / 1e9 / peak if loop_ms else None}
    ingest_bytes = (4 * F + 4 * V + F + 1) * N
    select_bytes = (4 * F + 4) * N
    train_ms = ms - step_ms_phases.get("select", 0)
    step_frac = {"survey_bytes_per_step": ingest_bytes + loop_bytes + select_bytes,
                 "frac": (ingest_bytes + loop_bytes + select_bytes) / (ms / 1e3) / 1e9 / peak,
                 "train_frac": (ingest_bytes + loop_bytes) / (train_ms / 1e3) / 1e9 / peak,
                 "rule": "SURVEY 8(d) bytes of the whole step (ingest + (F+1) per active row per level "
                         "+ select) / step time / peak; train_frac without the select"}
    cpu = None
    if world == 1 and not args.no_cpu:
        rows = {"C4": 1_500_000, "C3": 1_000_000}.get(args.config, N)  # ~20 s of oracle work
        cores, model_name = host_cpu()
        v, dt = cpu_baseline(cfg, min(rows, N), cfg.D)
        va, dta = cpu_baseline(cfg, min(rows, N), cfg.D, omp=True)
        cpu = {"value": v, "unit": "samples/s", "cores": 1, "kind": "oracle",
               "sample": f"first {min(rows, N)} rows of {args.config}: labels + depth-{cfg.D} exact "
                         f"CART + select, single-threaded C oracle ({dt:.1f} s)",
               "host_cores": cores, "cpu_model": model_name,
               "all_cores": {"value": va, "unit": "samples/s", "cores": cores,
                             "sample": f"same sample, liboracle_omp.so (oracle.c with -fopenmp: "
                                       f"features of a node and vectors in parallel) ({dta:.1f} s)"}}
        if args.config == "C4" and not args.no_c2:  # the small configs, whole tables
            per = {}
            for name, omp in (("C1", False), ("C2", False), ("C3", True)):
                c = synth.CONFIGS[name]
                rows_c = c.N if c.regions == 1 else len(synth.region_rows(c, 0))
                vc, dtc = cpu_baseline(c, rows_c, c.D, omp=omp)
                per[name] = {"value": vc, "unit": "samples/s", "seconds": dtc, "rows": rows_c,
                             "cores": cores if omp else 1,
                             "sample": f"first {rows_c} rows of {name}: labels + depth-{c.D} CART + "
                                       f"select, {'all-cores' if omp else 'single-threaded'} oracle"}
            cpu["per_config"] = per
    line = {
        "metric": METRIC, "value": N / (ms / 1e3), "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "rows": N, "features": cfg.F,
                   "variants": cfg.V, "depth": cfg.D, "model": model, "select_vectors": N,
                   "parallelism": f"dp{world}",
                   "l2": "inputs (%.1f GB) exceed the 126 MB L2; no flush needed" %
                         (N * 4 * (cfg.F + cfg.V) / 1e9)},
        "train_samples_per_s": N / (train_ms / 1e3),
        "select_per_s": N / (step_ms_phases["select"] / 1e3) if step_ms_phases.get("select") else None,
        "hbm_frac_step": step_frac,
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": int(round(sum(v["launches"] for v in kern.values()) / prof_steps * args.steps)),
        "gpu_launches_per_step": sum(v["launches"] for v in kern.values()) / prof_steps,
        "gpu_launches_rule": "the library's own kernel launches per step (a counter bumped at every "
                             "launch site), counted over separate profiled steps, x the timed steps",
        "roofline": roofline,
        "level_loop_roofline": level_loop,
        "cpu_baseline": cpu,
        "record_path": rec,
        "select_c5": c5,
        "kfold": kfold,
        "c2_regions": c2,
        "c1_latency": c1,
        "c3_train": c3,
        "strong_scaling_proxy": proxy,
        "phase_ms_per_step": step_ms_phases,
        "tree_nodes": int(len(tree)),
        "levels": levels,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
