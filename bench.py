"""Benchmark of the stream-segment-tree hot path on B200 (BASELINE.json metric:
range-Tucker queries/sec & appended slices/sec, with roofline fractions).

Workload (config.workload, default "c2" = BASELINE.json configs[1]): series
(T=32768, 376, 6) fp64, ranks (10,10,4), leaf block 128, 1000 range queries of
length U[64, T]. One step = build the tree from scratch (burst append of all T
slices: 256 batched leaf ALS + 255 stitches, level-synchronous) and answer the
1000-query batch. Series and outputs are HBM-resident for `value`; `e2e` runs
the same step through the public API with pinned host buffers (H2D of the
slices and D2H of every query result inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

Multi-GPU (torchrun): every rank builds its own replica and answers its own
query shard (independent seeds) — the path shards with no data-path
collective ("scaling": "weak"); times are max over ranks via NCCL all-reduce.
--impl reference times the CPU restatement of the reference (oracle/, the
reference itself cannot be built here) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def query_outputs(eng, w, ranges, alloc):
    """TTQueryOut array pointing into one flat buffer from alloc(n_doubles)."""
    from paper_2501_06647_b200.tucktree import TTQueryOut, TTRange, dptr

    p = len(w.ranks)
    sizes = []
    for ts, te in ranges:
        L = int(te - ts)
        rc = [min(w.ranks[0], L)] + [min(r, d) for r, d in zip(w.ranks[1:], w.shape[1:])]
        rows = [L] + list(w.shape[1:])
        sizes.append([int(np.prod(rc))] + [rows[m] * rc[m] for m in range(p)])
    total = sum(sum(s) for s in sizes)
    buf, base = alloc(total)
    outs = (TTQueryOut * len(ranges))()
    rr = (TTRange * len(ranges))()
    off = 0
    for i, (ts, te) in enumerate(ranges):
        rr[i].ts, rr[i].te = int(ts), int(te)
        outs[i].core = C.cast(C.c_void_p(base + 8 * off), dptr)
        off += sizes[i][0]
        for m in range(p):
            outs[i].factors[m] = C.cast(C.c_void_p(base + 8 * off), dptr)
            off += sizes[i][1 + m]
    return buf, outs, rr, total * 8


def query_algorithmic_bytes(w, tree, ranges):
    """hit temporal rows + hit factors/cores + outputs, per query."""
    p = len(w.ranks)
    nt = sum(d * r for d, r in zip(w.shape[1:], w.ranks[1:]))
    pr = int(np.prod(w.ranks))
    total = 0
    for ts, te in ranges:
        hits = tree.recall(int(ts), int(te))
        s = len(hits)
        rows = sum((h.end - h.begin) * w.ranks[0] for h in hits)
        L = int(te - ts)
        total += 8 * (rows + s * (nt + pr) + L * min(w.ranks[0], L) + nt + pr)
    return total


def run_engine(args, rank, world, local_rank):
    import torch

    import paper_2501_06647_b200 as eng
    from paper_2501_06647_b200 import synth

    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = synth.CONFIGS[args.config]
    T = w.shape[0]
    nq = args.queries or w.n_queries
    x = synth.generate(w, seed=0)
    ranges = synth.ranges(w, T, nq, seed=1 + rank)
    L = eng.lib()
    xd = torch.from_numpy(x).to(dev)
    xh = torch.from_numpy(x).pin_memory()

    def dev_alloc(n):
        t = torch.empty(n, dtype=torch.float64, device=dev)
        return t, t.data_ptr()

    def host_alloc(n):
        t = torch.empty(n, dtype=torch.float64).pin_memory()
        return t, t.data_ptr()

    dbuf, douts, rr, out_bytes = query_outputs(eng, w, ranges, dev_alloc)
    hbuf, houts, _, _ = query_outputs(eng, w, ranges, host_alloc)
    nsteps = args.warmup + args.steps
    mk = lambda: eng.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=w.leaf_block, device=local_rank)
    tree_v, tree_e = mk(), mk()  # each step clears and rebuilds (buffers kept: no allocation in the timed region)
    trees = [tree_v] * nsteps
    e2e_trees = [tree_e] * nsteps
    torch.cuda.synchronize()

    def step(tree, device_resident):
        tree.clear()
        if device_resident:
            tree.append_device(xd.data_ptr(), T)
        else:
            eng.tucktree._check(L.tt_append(tree._h, C.cast(C.c_void_p(xh.data_ptr()), eng.tucktree.dptr), T, 0))
        ta = tree.last_timing_ms()
        outs = douts if device_resident else houts
        eng.tucktree._check(L.tt_query_batch(tree._h, rr, nq, float("nan"), outs, 1 if device_resident else 0))
        tq = tree.last_timing_ms()
        return ta, tq

    # ---------------- device-resident (value) ----------------
    for i in range(args.warmup):
        step(trees[i], True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.kernel_launches()
    stats0 = eng.solver_stats()
    t_app = t_q = t_leaf = t_stitch_build = t_stitch_q = 0.0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record()
        for i in range(args.warmup, nsteps):
            ta, tq = step(trees[i], True)
            t_app += ta[2]
            t_leaf += ta[0]
            t_stitch_build += ta[1]
            t_q += tq[2]
            t_stitch_q += tq[1]
        ev1.record()
        torch.cuda.synchronize()
    launches = eng.kernel_launches() - launches0
    stats1 = eng.solver_stats()
    solver = {k: (stats1[k] - stats0[k]) / args.steps for k in ("problems", "als_sweeps", "eig_calls", "jacobi_sweeps",
                                                                "subspace_ok", "subspace_fallback", "subspace_iters")}
    span_ms = ev0.elapsed_time(ev1)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    # ---------------- end to end through the public API ----------------
    for i in range(args.warmup):
        step(e2e_trees[i], False)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2 = torch.cuda.Event(enable_timing=True)
    e2e_app = e2e_q = 0.0
    for i in range(args.warmup, nsteps):
        e0.record()
        tr = e2e_trees[i]
        tr.clear()
        eng.tucktree._check(L.tt_append(tr._h, C.cast(C.c_void_p(xh.data_ptr()), eng.tucktree.dptr), T, 0))
        e1.record()
        eng.tucktree._check(L.tt_query_batch(tr._h, rr, nq, float("nan"), houts, 0))
        e2.record()
        torch.cuda.synchronize()
        e2e_app += e0.elapsed_time(e1)
        e2e_q += e1.elapsed_time(e2)

    vals = torch.tensor([t_app, t_q, span_ms, e2e_app, e2e_q, t_leaf, t_stitch_q], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    t_app, t_q, span_ms, e2e_app, e2e_q, t_leaf, t_stitch_q = [float(v) for v in vals.tolist()]
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    K = args.steps
    qps = world * nq * K / (t_q / 1e3)
    sps = world * T * K / (t_app / 1e3)
    e2e_qps = world * nq * K / (e2e_q / 1e3)
    e2e_sps = world * T * K / (e2e_app / 1e3)
    peak, peak_kind = _peaks()
    # roofline of the dominant kernel (by device time in the step)
    leaf_bytes = x.nbytes  # one launch decomposes every leaf block; X read once is the algorithmic minimum
    leaf_gbs = leaf_bytes * K / (t_leaf / 1e3) / 1e9
    qbytes = query_algorithmic_bytes(w, trees[-1], ranges)
    q_gbs = qbytes * K / (t_stitch_q / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof))
        except Exception:
            traffic = None
    if t_stitch_q >= t_leaf:
        roof = {"kernel": "stitch_als_kernel (range-query batch)", "bound": "hbm", "achieved": round(q_gbs, 3),
                "peak": peak, "unit": "GB/s", "frac": round(q_gbs / peak, 5),
                "traffic": (traffic or {}).get("stitch_als_kernel"),
                "algorithmic_bytes_per_launch": qbytes, "peak_kind": peak_kind}
    else:
        roof = {"kernel": "leaf_als_kernel", "bound": "hbm", "achieved": round(leaf_gbs, 3), "peak": peak,
                "unit": "GB/s", "frac": round(leaf_gbs / peak, 5), "traffic": (traffic or {}).get("leaf_als_kernel"),
                "algorithmic_bytes_per_launch": leaf_bytes, "peak_kind": peak_kind}
    line = {
        "metric": "range_tucker_queries_per_s",
        "value": round(qps, 3),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(span_ms / K, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded; " + w.desc + ")",
        "config": {"workload": w.name, "shape": list(w.shape), "ranks": list(w.ranks), "leaf_block": w.leaf_block,
                   "queries_per_step": nq, "slices_per_step": T, "series_bytes": x.nbytes,
                   "l2": (f"inputs larger than L2 ({x.nbytes / 1e6:.0f} MB series re-read by every step's build)"
                          if x.nbytes > 126e6 else
                          f"series ({x.nbytes / 1e6:.0f} MB) fits the 126 MB L2: no flush between steps, so the "
                          "build may hit L2 (the C1 line is a parity/latency case, not the headline)"),
                   "step": "full tree build (burst append from HBM) + query batch"},
        "append": {"value": round(sps, 3), "unit": "slices/s", "ms_per_step": round(t_app / K, 4)},
        "phases_ms_per_step": {"append": round(t_app / K, 4), "append_leaf_als": round(t_leaf / K, 4),
                               "queries": round(t_q / K, 4), "queries_stitch": round(t_stitch_q / K, 4)},
        "e2e": {"value": round(e2e_qps, 3), "unit": "queries/s", "h2d_bytes_per_step": int(x.nbytes),
                "d2h_bytes_per_step": int(out_bytes), "append_slices_per_s": round(e2e_sps, 3)},
        "roofline": roof,
        "gpu_launches": int(launches),
        "solver_per_step": solver,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, x, ranges, args)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_baseline(w, x, ranges, args):
    """Oracle (CPU restatement of the reference) on the host cores: full tree
    build single-threaded (reference-faithful), then a query sample split over
    all cores (the reference's read-only concurrency contract)."""
    from oracle import oracle as O

    O.set_threads(1)
    T = w.shape[0]
    tr = O.Tree(w.shape[1:], w.ranks, leaf_block=w.leaf_block)
    t0 = time.perf_counter()
    tr.append(x)
    build_s = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    n = min(len(ranges), args.cpu_queries)
    t0 = time.perf_counter()
    tr.query_batch_checksums(ranges[:n], threads=cores)
    q_s = time.perf_counter() - t0
    return {"value": round(n / q_s, 3), "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": f"oracle build of all {T} slices on 1 thread ({build_s:.1f} s, {T / build_s:.1f} slices/s), "
                      f"then the first {n} of the step's queries over {cores} threads ({q_s:.1f} s)",
            "append_slices_per_s": round(T / build_s, 3)}


def run_reference(args, rank, world):
    """--impl reference: the CPU restatement timed on this host's cores."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2501_06647_b200 import synth

    w = synth.CONFIGS[args.config]
    T = w.shape[0]
    x = synth.generate(w, seed=0)
    ranges = synth.ranges(w, T, w.n_queries, seed=1)
    O.set_threads(1)
    tr = O.Tree(w.shape[1:], w.ranks, leaf_block=w.leaf_block)
    t0 = time.perf_counter()
    tr.append(x)
    build_s = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    per = args.ref_queries
    for i in range(args.warmup):
        tr.query_batch_checksums(ranges[(i * per) % len(ranges):][:per], threads=cores)
    times = []
    for i in range(args.steps):
        sl = ranges[((args.warmup + i) * per) % len(ranges):][:per]
        t0 = time.perf_counter()
        tr.query_batch_checksums(sl, threads=cores)
        times.append(time.perf_counter() - t0)
    q_s = sum(times)
    qps = per * args.steps / q_s
    sample = (f"per step {per} of the workload's queries over {cores} threads on the oracle tree; tree built once "
              f"from all {T} slices on 1 thread in {build_s:.1f} s")
    line = {
        "metric": "range_tucker_queries_per_s", "value": round(qps, 3), "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * q_s / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; " + w.desc + ")",
        "config": {"workload": w.name, "shape": list(w.shape), "ranks": list(w.ranks), "leaf_block": w.leaf_block,
                   "queries_per_step": per},
        "impl": "reference",
        "append": {"value": round(T / build_s, 3), "unit": "slices/s"},
        "cpu_baseline": {"value": round(qps, 3), "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(qps, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--queries", type=int, default=0)
    ap.add_argument("--cpu-queries", type=int, default=64)
    ap.add_argument("--ref-queries", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_engine(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
