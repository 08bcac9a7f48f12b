"""Benchmark of the stream-segment-tree hot path on B200 (BASELINE.json metric:
range-Tucker queries/sec & appended slices/sec, with roofline fractions).

Default workload = BASELINE.json configs[2] (C3), the largest configuration
that fits one GPU (5.77 GB series), in its BASELINE form: series
(T=16384, 500, 88) fp64 with Student-t(df=3) entries on a rank-(10,10,10)
backbone, leaf block 64; the tree is built from the first 12288 slices
(setup, reported as "build"), then slices are appended ONE AT A TIME with one
range query over the current [0, T) after every 16 appends.
One step = one leaf block of the stream: 64 single-slice appends + 4 queries
(the append that completes the block runs the leaf ALS and its stitch chain).
`value` = queries/s of that interleaved stream (slices, resident in HBM, are
appended from device memory; query outputs land in device buffers);
`append.value` = streamed slices/s of the same run; `e2e` = the same stream
through the public C ABI from pinned HOST slices with HOST query outputs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
                  [--config c1|c2|c3|c4] [--form stream|burst]

--form burst (default for C1/C2/C4) is the round-1 step: build the whole tree
from HBM in one burst append, then one batched query launch.
Multi-GPU (torchrun): every rank runs an independent replica on its own seeded
series (no data-path collective, "scaling": "weak"); times are max over ranks.
--impl reference times the CPU restatement of the reference (oracle/, pinned to
the reference's own sources by tests/test_ref_pin.py) on the host cores.
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
    x = synth.generate(w, seed=rank)  # independent replica per rank (weak scaling counts distinct work)
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
    sp0 = eng.stream_pass_stats()
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
    sp1 = eng.stream_pass_stats()
    step_pass = {k: sp1[k] - sp0[k] for k in sp0}
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
    traffic = load_traffic(w.name)  # ncu captures are keyed by workload; null without one for this workload
    if t_stitch_q >= t_leaf:
        roof = {"kernel": "stitch_als_kernel (range-query batch)", "bound": "hbm", "achieved": round(q_gbs, 3),
                "peak": peak, "unit": "GB/s", "frac": round(q_gbs / peak, 5),
                "traffic": traffic.get("stitch"),
                "algorithmic_bytes_per_launch": qbytes, "peak_kind": peak_kind}
    else:
        roof = {"kernel": "leaf ALS of the build (grid_ttm passes + per-leaf solver kernels)", "bound": "hbm",
                "achieved": round(leaf_gbs, 3), "peak": peak,
                "unit": "GB/s", "frac": round(leaf_gbs / peak, 5), "traffic": traffic.get("leaf"),
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
        "stream_pass": pass_roof(step_pass, {"launches": 0, "ms": 0.0, "bytes": 0.0}, peak, {}),
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


def run_engine_sharded(args, rank, world, local_rank):
    """--form burst at N > 1: the SURVEY §8(e) partitioning. Each rank builds the
    subtree of its leaf run from its own slices (no raw data moves), the node
    payloads are NCCL all-gathered and the top log2(N) levels stitched, then
    the query batch is split by cost and only the small results are gathered.
    Total work is fixed as N grows ("scaling": "strong")."""
    import torch
    import torch.distributed as dist

    import paper_2501_06647_b200 as eng
    from paper_2501_06647_b200 import distributed as D
    from paper_2501_06647_b200 import shard, synth

    if world == 1:  # --sharded without torchrun: a world of one
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = synth.CONFIGS[args.config]
    T = w.shape[0]
    nq = args.queries or w.n_queries
    B = w.leaf_block
    T = (T // B) * B
    plan = shard.plan_build(T // B, world)
    lo, hi = D.run_of(plan[rank], B)
    xd = synth.generate_torch(w, seed=0, T=T, device=dev)  # one series; each rank reads only its run
    ranges = synth.ranges(w, T, nq, seed=1)
    be = D.EngineBackend(w.shape[1:], w.ranks, B, device=local_rank)
    ss = int(np.prod(w.shape[1:]))

    def step():
        tree, gs, st = D.build_sharded(be, xd.data_ptr() + 8 * lo * ss, T, plan, rank, dev, on_device=True)
        torch.cuda.synchronize()
        tb = time.perf_counter()
        res, u0 = D.query_sharded(be, tree, ranges, rank, world, dev)
        torch.cuda.synchronize()
        return st, time.perf_counter() - tb

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.kernel_launches()
    tq = 0.0
    with ClockSampler(local_rank) as clk:
        ev0.record()
        for _ in range(args.steps):
            st, dq = step()
            tq += dq
        ev1.record()
        torch.cuda.synchronize()
    span = ev0.elapsed_time(ev1)
    launches = eng.kernel_launches() - launches0
    vals = torch.tensor([span, tq * 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    span, tq_ms = [float(v) for v in vals.tolist()]
    if rank == 0:
        K = args.steps
        line = {
            "metric": "range_tucker_queries_per_s", "value": round(nq * K / (tq_ms / 1e3), 3), "unit": "queries/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": round(span / K, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; " + w.desc + ")",
            "config": {"workload": w.name + "_sharded", "shape": [T] + list(w.shape[1:]), "ranks": list(w.ranks),
                       "leaf_block": B, "queries_per_step": nq, "slices_per_step": T,
                       "parallelism": f"node-partitioned build over {world} ranks + cost-split query batch",
                       "step": "sharded build (local subtrees, NCCL all-gather of node payloads, top stitches, "
                               "tree install) + sharded query batch (NCCL all-gather of the small results)"},
            "append": {"value": round(T * K / (span / 1e3), 3), "unit": "slices/s (whole step)"},
            "build_stats": st,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# ---------------------------------------------------------------------------
# Streaming form (BASELINE C3): single-slice appends with interleaved queries.
def stream_layout(w, steps_total):
    """(T0, block, per_query, T_series): the series is the config's T unless
    more steps than its 4096 streamed slices are asked for."""
    B = w.leaf_block
    T0 = w.build_T
    need = T0 + B * steps_total
    return T0, B, 16, max(w.shape[0], need)


def stream_alg_bytes(w, T_hits, hits, L):
    """SURVEY §8(d)(c) algorithmic bytes of one query given its hit list."""
    nt = sum(d * r for d, r in zip(w.shape[1:], w.ranks[1:]))
    pr = int(np.prod(w.ranks))
    rows = sum((h.end - h.begin) * w.ranks[0] for h in hits)
    return 8 * (rows + len(hits) * (nt + pr) + L * min(w.ranks[0], L) + nt + pr)


def run_engine_stream(args, rank, world, local_rank):
    import torch

    import paper_2501_06647_b200 as eng
    from paper_2501_06647_b200 import synth
    from paper_2501_06647_b200.tucktree import TTQueryOut, TTRange, dptr

    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = synth.CONFIGS[args.config]
    K, Wm = args.steps, args.warmup
    T0, B, every, Tser = stream_layout(w, K + Wm)
    # the series is generated on the device (the 5.8 GB numpy path takes ~1 min);
    # only the streamed slices are staged in pinned host memory for e2e
    xd = synth.generate_torch(w, seed=rank, T=Tser, device=dev)  # independent replica per rank
    ss = int(np.prod(w.shape[1:]))
    p = len(w.ranks)
    L = eng.lib()
    xh = xd[T0:].cpu().pin_memory()
    r0 = w.ranks[0]
    rc = [min(r, d) for r, d in zip(w.ranks[1:], w.shape[1:])]
    out_n = int(np.prod(w.ranks)) + Tser * r0 + sum(d * r for d, r in zip(w.shape[1:], rc))
    dq = torch.empty(out_n, dtype=torch.float64, device=dev)
    hq = torch.empty(out_n, dtype=torch.float64).pin_memory()

    def outs_for(buf, Tn):
        o = TTQueryOut()
        base = buf.data_ptr()
        o.core = C.cast(C.c_void_p(base), dptr)
        off = int(np.prod(w.ranks))
        o.factors[0] = C.cast(C.c_void_p(base + 8 * off), dptr)
        off += Tn * r0
        for m in range(1, p):
            o.factors[m] = C.cast(C.c_void_p(base + 8 * off), dptr)
            off += w.shape[m] * rc[m - 1]
        return o, 8 * (int(np.prod(w.ranks)) + Tn * min(r0, Tn) + sum(d * r for d, r in zip(w.shape[1:], rc)))

    mk = lambda: eng.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=B, device=local_rank)
    tree, tree_e = mk(), mk()
    # ---- setup: burst build of the first T0 slices (timed separately as "build");
    # one untimed build on a scratch tree first, so kernel loading, shared-memory
    # attributes and workspace growth are not in the timed build
    warm = mk()
    warm.append_device(xd.data_ptr(), T0)
    del warm
    torch.cuda.synchronize()
    sp0 = eng.stream_pass_stats()
    b0 = time.perf_counter()
    tree.append_device(xd.data_ptr(), T0)
    build_s = time.perf_counter() - b0
    build_ms = tree.last_timing_ms()
    sp1 = eng.stream_pass_stats()
    build_pass = {k: sp1[k] - sp0[k] for k in sp0}
    tree_e.append_device(xd.data_ptr(), T0)
    torch.cuda.synchronize()
    acc = {"leaf": 0.0, "stitch": 0.0, "tail": 0.0, "qstitch": 0.0}
    lat_app, lat_leafapp, lat_q = [], [], []
    alg = {"leaf": 0, "stitch": 0}
    nleaf = [0]

    def stream_step(tr, c, where, buf, record):
        """One leaf block: B single-slice appends, a [0, T) query every `every`."""
        Tcur = tr.timespan()
        for j in range(B):
            t = Tcur + j
            if where == 1:
                src = C.cast(C.c_void_p(xd.data_ptr() + 8 * t * ss), dptr)
            else:
                src = C.cast(C.c_void_p(xh.data_ptr() + 8 * (t - T0) * ss), dptr)
            a0 = time.perf_counter()
            eng.tucktree._check(L.tt_append(tr._h, src, 1, where))
            da = time.perf_counter() - a0
            if record:
                ms = tr.last_timing_ms()
                done_leaf = (t + 1) % B == 0
                lat_app.append(da)
                if done_leaf:
                    lat_leafapp.append(da)
                    acc["leaf"] += ms[0]
                    acc["stitch"] += ms[1]
                    nleaf[0] += 1
                    alg["leaf"] += 8 * B * ss
                    # stitch chain: parent lengths 2B, 4B, ... while the node completes
                    lv, li = 1, (t + 1) // B
                    while li % (1 << lv) == 0:
                        Lp = B << lv
                        # two children's rows + factors + cores read, the parent's L x r0 written
                        nt_pr = sum(d * r for d, r in zip(w.shape[1:], rc)) + int(np.prod(w.ranks))
                        alg["stitch"] += 8 * (Lp * r0 + 2 * nt_pr + Lp * r0)
                        lv += 1
            if (j + 1) % every == 0:
                Tn = t + 1
                rr = TTRange()
                rr.ts, rr.te = 0, Tn
                o, ob = outs_for(buf, Tn)
                q0 = time.perf_counter()
                eng.tucktree._check(L.tt_query_batch(tr._h, C.byref(rr), 1, float("nan"), C.byref(o), where))
                dq_ = time.perf_counter() - q0
                if record:
                    ms = tr.last_timing_ms()
                    lat_q.append(dq_)
                    acc["tail"] += ms[0]
                    acc["qstitch"] += ms[1]
                    hits = tr.recall(0, Tn)
                    alg["stitch"] += stream_alg_bytes(w, Tn, [h for h in hits if h.flag != 2], Tn)
                    alg["leaf"] += 8 * sum(h.end - h.begin for h in hits if h.flag == 2) * ss

    # ---------------- device-resident (value) ----------------
    for c in range(Wm):
        stream_step(tree, c, 1, dq, False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.kernel_launches()
    stats0 = eng.solver_stats()
    sp0 = eng.stream_pass_stats()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record()
        for c in range(K):
            stream_step(tree, Wm + c, 1, dq, True)
        ev1.record()
        torch.cuda.synchronize()
    span_ms = ev0.elapsed_time(ev1)
    launches = eng.kernel_launches() - launches0
    sp1 = eng.stream_pass_stats()
    step_pass = {k: sp1[k] - sp0[k] for k in sp0}
    stats1 = eng.solver_stats()
    solver = {k: (stats1[k] - stats0[k]) / K for k in ("problems", "als_sweeps", "eig_calls", "jacobi_sweeps",
                                                       "subspace_ok", "subspace_fallback", "subspace_iters")}
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # ---------------- end to end: pinned host slices in, host outputs out ----------------
    for c in range(Wm):
        stream_step(tree_e, c, 0, hq, False)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for c in range(K):
        stream_step(tree_e, Wm + c, 0, hq, False)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    vals = torch.tensor([span_ms, e2e_ms, acc["leaf"], acc["stitch"], acc["tail"], acc["qstitch"]],
                        dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    span_ms, e2e_ms, t_leaf, t_stitch, t_tail, t_qstitch = [float(v) for v in vals.tolist()]
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    nq = K * (B // every)
    qps = world * nq / (span_ms / 1e3)
    sps = world * K * B / (span_ms / 1e3)
    peak, peak_kind = _peaks()
    t_leafk = t_leaf + t_tail
    t_stk = t_stitch + t_qstitch
    traffic = load_traffic(w.name + "_stream")
    if t_stk >= t_leafk:
        gbs = alg["stitch"] / (t_stk / 1e3) / 1e9
        roof = {"kernel": "stitch_als_kernel (append stitch chains + [0,T) query stitches)", "bound": "hbm",
                "achieved": round(gbs, 3), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 6),
                "traffic": traffic.get("stitch"), "algorithmic_bytes_per_step": alg["stitch"] // K,
                "peak_kind": peak_kind}
    else:
        gbs = alg["leaf"] / (t_leafk / 1e3) / 1e9
        roof = {"kernel": "grid-wide leaf ALS (grid_ttm/grid_last/grid_gram + grid_solve kernels: streamed leaf "
                          "blocks + query tails)", "bound": "hbm",
                "achieved": round(gbs, 3), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 6),
                "traffic": traffic.get("leaf"), "algorithmic_bytes_per_step": alg["leaf"] // K,
                "peak_kind": peak_kind}
    la, ll, lq = (np.array(v) * 1e3 for v in (lat_app, lat_leafapp, lat_q))
    q_out_bytes = sum(outs_for(dq, T0 + Wm * B + c * B + (j + 1) * every)[1] for c in range(K) for j in range(B // every))
    build_gbs = 8 * T0 * ss / (build_ms[0] / 1e3) / 1e9 if build_ms[0] > 0 else None
    line = {
        "metric": "range_tucker_queries_per_s",
        "value": round(qps, 3),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": K,
        "warmup": Wm,
        "ms_per_step": round(span_ms / K, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded; " + w.desc + ")",
        "config": {"workload": w.name + "_stream", "shape": [Tser] + list(w.shape[1:]), "ranks": list(w.ranks),
                   "leaf_block": B, "build_slices": T0, "slices_per_step": B, "queries_per_step": B // every,
                   "query": "[0, T) over the current timespan after every 16th single-slice append",
                   "l2": "inputs larger than L2 (the 5.8 GB series streams slice by slice; every leaf block and "
                         "query tail is read from HBM the first time it is touched)",
                   "step": "64 single-slice appends from HBM (one completes a leaf block: leaf ALS + stitch chain) "
                           "+ 4 range queries [0, T)"},
        "append": {"value": round(sps, 3), "unit": "slices/s", "latency_ms": {
            "p50": round(float(np.median(la)), 4), "p99": round(float(np.percentile(la, 99)), 4),
            "block_completing_p50": round(float(np.median(ll)), 4),
            "block_completing_p99": round(float(np.percentile(ll, 99)), 4),
            "block_completing_max": round(float(ll.max()), 4)}},
        "query_latency_ms": {"p50": round(float(np.median(lq)), 4), "p99": round(float(np.percentile(lq, 99)), 4),
                             "max": round(float(lq.max()), 4)},
        "phases_ms_per_step": {"append_leaf_als": round(t_leaf / K, 4), "append_stitch_chain": round(t_stitch / K, 4),
                               "query_tail_als": round(t_tail / K, 4), "query_stitch": round(t_qstitch / K, 4),
                               "host_and_sync": round((span_ms - t_leaf - t_stitch - t_tail - t_qstitch) / K, 4)},
        "build": {"slices": T0, "slices_per_s": round(T0 / build_s, 1), "device_ms": round(float(build_ms[2]), 3),
                  "leaf_phase_ms": round(float(build_ms[0]), 3), "stitch_phase_ms": round(float(build_ms[1]), 3),
                  "leaf_phase_gbs": round(build_gbs, 2) if build_gbs else None,
                  "leaf_phase_frac": round(build_gbs / peak, 5) if build_gbs else None},
        "e2e": {"value": round(world * nq / (e2e_ms / 1e3), 3), "unit": "queries/s",
                "h2d_bytes_per_step": int(B * ss * 8), "d2h_bytes_per_step": int(q_out_bytes // K),
                "append_slices_per_s": round(world * K * B / (e2e_ms / 1e3), 3)},
        "roofline": roof,
        "stream_pass": pass_roof(step_pass, build_pass, peak, traffic),
        "gpu_launches": int(launches),
        "solver_per_step": solver,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_stream_sample(w, xh.numpy(), T0, args)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def pass_roof(step_pass, build_pass, peak, traffic):
    """Achieved HBM bandwidth of grid_ttm_kernel's passes over X (the only kernel
    of the path that moves leaf-block-sized data), from the engine's CUDA events
    around each launch: inside the timed steps (one leaf block or query tail per
    launch, L2-resident after the first pass) and in the 192-leaf build
    (4.3 GB per launch, from HBM)."""
    out = {"kernel": "grid_ttm_kernel (X x_1 U_1^T and X x_0 U_0^T passes)", "bound": "hbm", "unit": "GB/s", "peak": peak}
    for tag, sp in (("steps", step_pass), ("build", build_pass)):
        if sp["launches"] > 0 and sp["ms"] > 0:
            gbs = sp["bytes"] / (sp["ms"] / 1e3) / 1e9
            out[tag] = {"launches": int(sp["launches"]), "avg_launch_ms": round(sp["ms"] / sp["launches"], 4),
                        "bytes_per_launch": int(sp["bytes"] / sp["launches"]), "achieved": round(gbs, 1),
                        "frac": round(gbs / peak, 4)}
    if "build" in out:  # ncu dram__bytes_read+write of one build-sized launch (profiles/traffic.json), or null
        out["build"]["traffic"] = traffic.get("stream_pass_build")
    return out


def load_traffic(key):
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(prof))
        v = t.get(key)
        return v if isinstance(v, dict) else {}
    except Exception:
        return {}


def _synthetic_node(rng, L, w, ref):
    """A stored-node-shaped part (L-row temporal factor, the config's non-temporal
    factors, full core) for timing the CPU stitch: cost depends on shapes only."""
    from oracle import oracle as O

    q, _ = np.linalg.qr(rng.standard_normal((L, min(w.ranks[0], L))))
    core = rng.standard_normal([q.shape[1]] + [ref.rank(m) for m in range(1, len(w.ranks))])
    return O.Factors(core, [q] + [ref.factors[m] for m in range(1, len(w.ranks))])


def cpu_stream_cycle(w, xs, T0, c, threads, cache):
    """CPU time (s) of streaming cycle c on the oracle: the leaf ALS of the
    completed block, its stitch chain (two-part stitches of lengths 2B, 4B, ...)
    and the 4 [0, T) queries (tail ALS + stitch of the entire hits + tail)."""
    from oracle import oracle as O

    O.set_threads(threads)
    B = w.leaf_block
    rng = np.random.default_rng(c)
    t_start = time.perf_counter()
    li = T0 // B + c  # index of the leaf this cycle completes
    leaf = O.tucker_als(xs[li * B - T0:(li + 1) * B - T0], w.ranks)  # xs starts at slice T0
    cache.setdefault("leaf", leaf)
    lv = 1
    while (li + 1) % (1 << lv) == 0:
        Lp = B << lv
        parts = [_synthetic_node(rng, Lp // 2, w, leaf), _synthetic_node(rng, Lp // 2, w, leaf)]
        O.stitch(parts, w.ranks)
        lv += 1
    for j in range(B // 16):
        tail = 16 * (j + 1) if j + 1 < B // 16 else 0
        nb = li + (1 if tail == 0 else 0)  # complete leaves at this query
        parts = []
        if tail:
            Ts = (li) * B
            parts_tail = O.tucker_als(xs[Ts - T0:Ts - T0 + tail], w.ranks)
        else:
            parts_tail = None
        # entire hits of [0, nb*B): the binary decomposition of nb
        bit = 1 << max(nb.bit_length() - 1, 0)
        while bit:
            if nb & bit:
                parts.append(_synthetic_node(rng, bit * B, w, leaf))
            bit >>= 1
        if parts_tail is not None:
            parts.append(parts_tail)
        O.stitch(parts, w.ranks)
    return time.perf_counter() - t_start


def cpu_stream_sample(w, xs, T0, args):
    """cpu_baseline for the streaming form: the oracle on sampled cycles (single
    thread, reference-faithful) — leaf ALS, stitch chain and 4 queries each."""
    cache = {}
    picks = [0, 15, 31, 63][: max(1, args.cpu_cycles)]
    ts = [cpu_stream_cycle(w, xs, T0, c, 1, cache) for c in picks if (c + 1) * w.leaf_block <= xs.shape[0]]
    per = sum(ts) / len(ts)
    return {"value": round((w.leaf_block // 16) / per, 4), "unit": "queries/s", "cores": 1, "kind": "port",
            "sample": f"oracle (restated reference, 1 thread) on {len(ts)} sampled stream cycles {picks[:len(ts)]}: "
                      f"leaf ALS of the completed 64-slice block + its stitch chain + 4 [0, T) queries (tail ALS + "
                      f"stitch of the entire hits; hit nodes carry stored-node shapes), {per:.2f} s per cycle",
            "append_slices_per_s": round(w.leaf_block / per, 3)}


def run_reference_stream(args, rank, world):
    """--impl reference for the streaming form: each step = one stream cycle on
    the oracle with all host cores given to its BLAS."""
    if rank != 0:
        return
    from paper_2501_06647_b200 import synth

    w = synth.CONFIGS[args.config]
    K, Wm = args.steps, args.warmup
    T0, B, every, Tser = stream_layout(w, K + Wm)
    # same seeded series as the engine arm (generated with torch, on the GPU when
    # present — input synthesis only, outside every timed region); the CPU
    # works on the streamed slices
    import torch

    gdev = "cuda" if torch.cuda.is_available() else "cpu"
    xs = synth.generate_torch(w, seed=0, T=Tser, device=gdev)[T0:].cpu().numpy()
    cores = os.cpu_count() or 1
    cache = {}
    ncyc = (Tser - T0) // B
    for c in range(Wm):
        cpu_stream_cycle(w, xs, T0, c % ncyc, cores, cache)
    tot = 0.0
    for i in range(K):
        tot += cpu_stream_cycle(w, xs, T0, (Wm + i) % ncyc, cores, cache)
    qps = K * (B // every) / tot
    line = {
        "metric": "range_tucker_queries_per_s", "value": round(qps, 4), "unit": "queries/s", "n_gpus": world,
        "steps": K, "warmup": Wm, "ms_per_step": round(1e3 * tot / K, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; " + w.desc + ")",
        "config": {"workload": w.name + "_stream", "shape": [Tser] + list(w.shape[1:]), "ranks": list(w.ranks),
                   "leaf_block": B, "build_slices": T0, "slices_per_step": B, "queries_per_step": B // every},
        "impl": "reference",
        "append": {"value": round(K * B / tot, 3), "unit": "slices/s"},
        "cpu_baseline": {"value": round(qps, 4), "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"per step one stream cycle on the oracle (restated reference): leaf ALS of the "
                                   f"completed block, its stitch chain, 4 [0, T) queries; BLAS on {cores} threads"},
        "e2e": {"value": round(qps, 4), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--form", default="", choices=["", "stream", "burst"])
    ap.add_argument("--cpu-cycles", type=int, default=2)
    ap.add_argument("--sharded", action="store_true", help="burst form through the sharded path even at N = 1")
    ap.add_argument("--queries", type=int, default=0)
    ap.add_argument("--cpu-queries", type=int, default=64)
    ap.add_argument("--ref-queries", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    from paper_2501_06647_b200 import synth

    form = args.form or ("stream" if synth.CONFIGS[args.config].build_T else "burst")
    if args.impl == "reference":
        (run_reference_stream if form == "stream" else run_reference)(args, rank, world)
    else:
        if form == "stream":
            run_engine_stream(args, rank, world, local_rank)
        elif world > 1 or args.sharded:
            run_engine_sharded(args, rank, world, local_rank)
        else:
            run_engine(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
