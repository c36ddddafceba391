#!/usr/bin/env python
"""Benchmark: analytic marching of BASELINE.json configs[1] on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one complete march (every analytic cell reachable from the seeds)
of the configs[1] network: 3-(90x6)-1 ReLU SDF MLP, SAL geometric (sphere-SDF)
init, fp64, seeded with the reference's default trigger (64 dichotomy seeds,
rng_seed 0).  ``value`` = visited cells / device time with the network and the
seed points resident in HBM; ``e2e`` = the same through the public
``march(net, MarchConfig)`` call from host buffers (engine creation + weight
upload, seeding, marching, results back to host, sorted like the reference).
With N > 1 ranks (torchrun, one per GPU) states are sharded by hash ownership
and the frontier is exchanged with one NCCL all-to-all per round of BFS
iterations (paper_2106_10031_b200/distributed.py).

``--impl reference`` times the reference algorithm's CPU implementation (the C
oracle restatement; the reference itself is pure Python) on the host cores.
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

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

WORKLOAD = ("configs[1]: 3-(90x6)-1 ReLU SDF MLP, SAL geometric (sphere-SDF) init seed 0, fp64, "
            "64 dichotomy seeds (reference default MarchConfig), box [-1.2,1.2]^3")
METRIC = "analytic cells/sec (full march of configs[1])"


def workload_net():
    from paper_2106_10031_b200 import synth
    return synth.geometric_mlp([90] * 6, seed=0)


def _peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def flush_l2(buf):
    buf.fill_(1)   # 512 MiB write > 126 MB L2


def cpu_baseline_run(net, seeds, target_seconds=15.0, threads=None, max_cells=None):
    """Oracle (C restatement of the reference) on the host cores over a bounded sample."""
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import oracle
    threads = threads or os.cpu_count() or 1
    on = oracle.OracleNet(net)
    if max_cells is None:
        t = time.perf_counter()
        probe = oracle.march(net, seed_points=seeds, max_cells=3000, threads=threads, oracle_net=on)
        rate = probe.report["cells_visited"] / max(time.perf_counter() - t, 1e-6)
        max_cells = int(max(5000, min(rate * target_seconds, 10_000_000)))
    t = time.perf_counter()
    r = oracle.march(net, seed_points=seeds, max_cells=max_cells, threads=threads, oracle_net=on)
    dt = time.perf_counter() - t
    cells = r.report["cells_visited"]
    return {"value": cells / dt, "unit": "cells/s", "cores": threads, "kind": "port",
            "sample": f"first {cells} cells (max_cells cap) of the same 64-seed march, {dt:.1f} s, "
                      f"oracle/am_oracle.c with {threads} threads"}, max_cells


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host CPU (oracle port)."""
    if rank != 0:
        return
    from paper_2106_10031_b200.engine import Engine  # noqa: F401  (seeds via the CPU trigger below)
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import oracle
    net = workload_net()
    on = oracle.OracleNet(net)
    seeds = oracle.sample_seeds(on, 64, ((-1.2,) * 3, (1.2,) * 3), "dichotomy", 0)
    threads = os.cpu_count() or 1
    _, cap = cpu_baseline_run(net, seeds, target_seconds=8.0, threads=threads)
    for _ in range(args.warmup):
        oracle.march(net, seed_points=seeds, max_cells=cap, threads=threads, oracle_net=on)
    times, cells = [], 0
    for _ in range(args.steps):
        t = time.perf_counter()
        r = oracle.march(net, seed_points=seeds, max_cells=cap, threads=threads, oracle_net=on)
        times.append(time.perf_counter() - t)
        cells = r.report["cells_visited"]
    dt = float(np.mean(times))
    v = cells / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "cells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_cells": cells, "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": v, "unit": "cells/s", "cores": threads, "kind": "port",
                         "sample": f"first {cells} cells of the march per step (max_cells cap)"},
        "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seeds", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the capped configs[2] measurement")
    ap.add_argument("--deepsdf-cells", type=int, default=1_000_000)
    ap.add_argument("--no-deepsdf-full", dest="deepsdf_full", action="store_false",
                    help="skip the complete (uncapped) configs[2] march line in other_configs")
    ap.add_argument("--latent-cells", type=int, default=20_000)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    # AM_BENCH_SHARE_GPU=1 / AM_DIST_BACKEND=gloo: functional check of the multi-rank path on a
    # one-GPU box (ranks share the device; the timings of such a run are not measurements)
    if os.environ.get("AM_BENCH_SHARE_GPU") == "1":
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    if world > 1:
        backend = os.environ.get("AM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)

    from paper_2106_10031_b200 import marching
    from paper_2106_10031_b200.engine import Engine
    from paper_2106_10031_b200 import _native
    from paper_2106_10031_b200.seeding import sample_seeds

    net = workload_net()
    bbox = ((-1.2,) * 3, (1.2,) * 3)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    if world > 1:
        from paper_2106_10031_b200.distributed import ShardedMarcher
        sm = ShardedMarcher(net, bbox=bbox)
        seeds = sm.sample_seeds(args.seeds, rng_seed=0)
        run_once = lambda: sm.run(seeds)  # noqa: E731
        engine = sm.engine
        stream = sm.stream   # the engine and its exchange run on the marcher's stream
    else:
        engine = Engine(net, bbox=bbox)
        seeds = sample_seeds(engine, args.seeds, bbox, rng_seed=0)
        seeds_dev = torch.as_tensor(seeds, device=dev)

        def run_once():
            engine.reset()
            engine.seed(seeds_dev)
            return engine.run()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        run_once()
    torch.cuda.synchronize()

    # ----------------------------------------------------- device-timed steps
    lib = _native.load()
    st0 = engine.stats()
    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush_l2(flush)
            barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            waves = run_once()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1))
    clocks = clk.summary()
    st1 = engine.stats()
    counts = engine.counts()
    assert counts["overflow"] == 0, "cells exceeded the face solver's limits: the march is incomplete"
    cells_local = counts["cells"]
    t_local = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([t_local, float(cells_local)], dtype=torch.float64, device=dev)
        tmax = tt[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        csum = tt[1:].clone()
        dist.all_reduce(csum, op=dist.ReduceOp.SUM)
        t_step, cells = float(tmax.item()), int(csum.item())
    else:
        t_step, cells = t_local, cells_local
    value = cells / (t_step * 1e-3)
    launches = (st1["launches"] - st0["launches"]) / max(args.steps, 1)

    # ------------------------------------------------- kernel timing (roofline)
    # timing mode: every BFS iteration is cut by CUDA events on the engine's stream into contiguous
    # stages (take, compose, canonical insert, frontier, near lists, face solver, flip insert,
    # probe records) + the exact probe forwards, so the stages add up to the iterations' device
    # time; one extra march, not part of the timed steps.  (Ranks > 1: measured on rank 0's own
    # single-GPU engine -- the per-kernel figures do not depend on sharding.)
    if world > 1:
        tengine = Engine(net, bbox=bbox)
        tseeds = torch.as_tensor(seeds, device=dev)

        def trun():
            tengine.reset()
            tengine.seed(tseeds)
            return tengine.run()
    else:
        tengine, trun = engine, run_once
    tengine.set_timing(True)
    te0, te1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tstream = tengine.stream
    te0.record(tstream)
    trun()          # stats are reset by the engine at the start of every march
    te1.record(tstream)
    torch.cuda.synchronize()
    timed_total = te0.elapsed_time(te1)
    s1 = tengine.stats()
    kt = tengine.kernel_times()
    tengine.set_timing(False)
    overflow = tengine.counts()["overflow"]
    assert overflow == 0, f"{overflow} cells exceeded the face solver's limits"
    pk = np.zeros(2)
    _native.check(lib.am_bench_fp64_peak(local_rank, pk.ctypes.data), "am_bench_fp64_peak")
    hbm, hbm_src = _peaks()
    traffic = {}
    prof = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh)

    def traffic_of(name):
        t = traffic.get(name)
        if not isinstance(t, dict):
            return {"traffic": t}
        return {"traffic": t.get("dram_bytes_per_launch"), "traffic_launch": t.get("launch"),
                "traffic_algorithmic_bytes": t.get("algorithmic_bytes_per_launch")}
    ms = kt["ms"]
    stage_sum = sum(ms.values())
    kw8 = kt["kw"] * 8
    comp_ms = ms["compose"]
    # executed DMMA work: the composition steps taken from parents' rows (prefix reuse) excluded
    comp_flops = s1["flops_per_cell"] * kt["composed"] - s1.get("prefix_skipped_flops", 0.0)
    comp_tf = comp_flops / (comp_ms * 1e-3) / 1e12 if comp_ms else 0.0
    face_ms = ms["near"] + ms["face"]
    face_gbs = s1["face_bytes"] / (face_ms * 1e-3) / 1e9 if face_ms else 0.0
    # hash inserts: every candidate reads its key and probes a slot; every new entry writes its
    # key, hint, slot and queue entry
    ins_ms = ms["canonical_insert"] + ms["flip_insert"]
    ins_bytes = (kt["flips"] + kt["canonical"]) * (kw8 + 8) + kt["new_entries"] * (kw8 + 8 + 32 + 4)
    ins_gbs = ins_bytes / (ins_ms * 1e-3) / 1e9 if ins_ms else 0.0
    rec_ms = ms["probe_records"]
    rec_bytes = kt["probe_records"] * (4 + 4 + 24 + 4)
    rec_gbs = rec_bytes / (rec_ms * 1e-3) / 1e9 if rec_ms else 0.0
    kernels = {
        "compose_dmma": {"bound": "tensor", "achieved": comp_tf, "peak": float(pk[0]), "unit": "TFLOP/s",
                         "frac": comp_tf / pk[0] if pk[0] else None, "ms": comp_ms,
                         "peak_source": "measured fp64 DMMA microbenchmark (am_bench_fp64_peak)",
                         "kernels": "k_compose_narrow: gather + every layer + face head in one launch (plain "
                                    "nets of width <= 96; else k_gather_input + k_gemm_step x L + k_face_head)",
                         "algorithmic": "sum_l 2 n_l n_(l-1) 4 FLOP per composed cell", **traffic_of("compose")},
        "face_stage": {"bound": "hbm", "achieved": face_gbs, "peak": hbm, "unit": "GB/s",
                       "frac": face_gbs / hbm, "ms": face_ms, "ms_near": ms["near"], "ms_face": ms["face"],
                       "peak_source": hbm_src, "kernels": "k_near + k_face",
                       "algorithmic": "NB*32 + M*32 + KW*8 bytes per faced cell (planes, faces, key read once)",
                       **traffic_of("face")},
        "hash_insert": {"bound": "hbm", "achieved": ins_gbs, "peak": hbm, "unit": "GB/s",
                        "frac": ins_gbs / hbm, "ms": ins_ms, "ms_canonical": ms["canonical_insert"],
                        "ms_flips": ms["flip_insert"], "peak_source": hbm_src,
                        "kernels": "k_route_changed + k_hash_upsert (canonical keys), k_hash_upsert (flips)",
                        "algorithmic": "(KW*8 + 8) B per candidate + (KW*8 + 52) B per new entry",
                        "candidates": kt["flips"] + kt["canonical"], "new_entries": kt["new_entries"]},
        "probe_records": {"bound": "hbm", "achieved": rec_gbs, "peak": hbm, "unit": "GB/s", "frac": rec_gbs / hbm,
                          "ms": rec_ms, "records": kt["probe_records"], "kernels": "k_probe_records",
                          "algorithmic": "36 B per probe record (target, neuron, point, status)"},
        "probe_forward_dmma": {"ms": ms["probe_forward"], "probes": s1["probes"],
                               "kernels": "exact forwards of unvalidated probes (k_gemm_step<1,64> x L + heads)"},
        "take": {"ms": ms["take"]}, "frontier": {"ms": ms["frontier"]},
    }
    stages = {"ms": {k: round(v, 4) for k, v in ms.items()},
              "share": {k: round(v / stage_sum, 4) if stage_sum else None for k, v in ms.items()},
              "sum_ms": stage_sum, "timed_march_ms": timed_total, "iterations": kt["iterations"],
              "of_step_ms": {k: round(v / stage_sum * t_step, 4) if stage_sum else None for k, v in ms.items()},
              "note": "ms: a timing-mode march cut into contiguous stages by CUDA events on the engine stream "
                      "(sum_ms; timed_march_ms = that march's device time incl. the host syncs between its "
                      "iterations); of_step_ms attributes the graph-replayed ms_per_step by those shares (sums to "
                      "ms_per_step).  Timing mode breaks PDL overlap at every event, so sum_ms > ms_per_step."}
    rooflined = ("compose_dmma", "face_stage", "hash_insert", "probe_records")
    dominant = max(rooflined, key=lambda k: kernels[k]["ms"])
    roof = dict(kernels[dominant])
    roof["kernel"] = dominant

    # ------------------------------------------------------------------ e2e
    # the public call a user makes, from host buffers: march(net, cfg) (engine set-up + weight
    # upload, seeding, BFS, sorted results back to host) + MarchResult.welded_mesh() (GPU weld,
    # welded mesh back to host) = the end-to-end mesh time
    e2e = None
    if world == 1:
        cfg = marching.MarchConfig(seeds=args.seeds, rng_seed=0, bbox=bbox)
        # cold first call: no cached engine for the architecture, no memoised trigger samples
        from paper_2106_10031_b200 import seeding
        marching.clear_engine_cache()
        seeding._BLOCKS.clear()
        seeding._ROUNDS.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cold = marching.march(net, cfg)
        cold.welded_mesh()
        cold_ms = (time.perf_counter() - t0) * 1e3
        del cold
        # warm: engine cache and pinned host blocks, with the same result lifetimes as the timed
        # loop (the previous step's result is alive while the next one is produced)
        prev = None
        for _ in range(max(args.warmup, 2)):
            cur = marching.march(net, cfg)
            prev = (cur, cur.welded_mesh())
        del prev, cur
        e_times, m_times = [], []
        h2d = d2h = 0
        from paper_2106_10031_b200.network import to_blob
        for _ in range(max(3, min(args.steps, 10))):
            flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = marching.march(net, cfg)
            t1 = time.perf_counter()
            mesh = r.welded_mesh()
            t2 = time.perf_counter()
            e_times.append((t2 - t0) * 1e3)
            m_times.append((t1 - t0) * 1e3)
            blob = to_blob(net)
            # inputs: parameters (weights + padded copies), step/sub tables, the trigger's sample
            # points (64 per seed) and bisection pairs; the soup stays in HBM for the weld
            h2d = (2 * blob.params.nbytes + blob.steps.nbytes + blob.subs.nbytes + args.seeds * 64 * 3 * 8
                   + args.seeds * 2 * 3 * 8)
            # outputs: the sorted march result and the welded mesh
            d2h = (r.keys.nbytes + r.nverts.nbytes + r.verts.nbytes + r.edge_nrefs.nbytes + r.edge_refs.nbytes
                   + mesh.vertices.nbytes + mesh.face_off.nbytes + mesh.face_idx.nbytes)
        e_ms = float(np.mean(e_times))
        e2e = {"value": r.report.cells_visited / (e_ms * 1e-3), "unit": "cells/s", "ms_per_step": e_ms,
               "ms_steps": [round(x, 2) for x in e_times], "cold_first_call_ms": cold_ms,
               "mesh_time_s": e_ms * 1e-3, "march_only_ms": float(np.mean(m_times)),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "mesh": {"vertices": int(mesh.n_vertices), "faces": int(mesh.n_faces),
                        "dropped": int(mesh.dropped_faces)},
               "api": "paper_2106_10031_b200.march(net, MarchConfig(seeds=64)).welded_mesh() from host buffers, "
                      "wall clock (host-synchronous API)"}

    elif world > 1:
        # the multi-GPU public call on every rank, from host buffers: march_sharded(net, cfg) =
        # seeding, the sharded BFS with its all-to-all frontier exchange, and each rank's sorted
        # share of the result (its owned cells with their polygons) back to host; mesh time =
        # the slowest rank
        from paper_2106_10031_b200.distributed import march_sharded
        from paper_2106_10031_b200.network import to_blob
        cfg = marching.MarchConfig(seeds=args.seeds, rng_seed=0, bbox=bbox)
        for _ in range(max(args.warmup, 2)):
            r = march_sharded(net, cfg)
        del r
        e_times = []
        for _ in range(max(1, min(args.steps, 3))):
            flush_l2(flush)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            r = march_sharded(net, cfg)
            t1 = time.perf_counter()
            barrier()
            e_times.append((t1 - t0) * 1e3)
        blob = to_blob(net)
        h2d_l = (2 * blob.params.nbytes + blob.steps.nbytes + blob.subs.nbytes + args.seeds * 64 * 3 * 8
                 + args.seeds * 2 * 3 * 8)
        d2h_l = r.keys.nbytes + r.nverts.nbytes + r.verts.nbytes + r.edge_nrefs.nbytes + r.edge_refs.nbytes
        agg = torch.tensor([float(np.mean(e_times)), float(r.report.cells_visited), float(h2d_l), float(d2h_l)],
                           dtype=torch.float64, device=dev)
        emax = agg[:1].clone()
        dist.all_reduce(emax, op=dist.ReduceOp.MAX)
        esum = agg[1:].clone()
        dist.all_reduce(esum, op=dist.ReduceOp.SUM)
        e_ms = float(emax.item())
        e_cells, h2d, d2h = (float(x) for x in esum.tolist())
        e2e = {"value": e_cells / (e_ms * 1e-3), "unit": "cells/s", "ms_per_step": e_ms,
               "mesh_time_s": e_ms * 1e-3, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "cells": int(e_cells),
               "api": "paper_2106_10031_b200.distributed.march_sharded(net, MarchConfig(seeds=64)) on every "
                      "rank from host buffers (each rank's sorted owned cells + polygons to host; no weld), "
                      "wall clock, max over ranks"}

    # --------------------------------------- the largest MLP (configs[2]), capped sample
    others = {}
    if world == 1 and not args.no_extra:
        from paper_2106_10031_b200 import synth
        dnet = synth.deepsdf_mlp(512, 8, 4, seed=0)
        cap = args.deepsdf_cells
        deng = Engine(dnet, bbox=bbox, max_cells=cap)
        dseeds = torch.as_tensor(sample_seeds(deng, args.seeds, bbox, rng_seed=0), device=dev)

        def drun():
            deng.reset()
            deng.seed(dseeds)
            return deng.run()
        drun()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dw = drun()
        e1.record(stream)
        torch.cuda.synchronize()
        d_ms = e0.elapsed_time(e1)
        dcells = deng.counts()["cells"]
        deng.set_timing(True)
        drun()
        ds = deng.stats()
        deng.set_timing(False)
        dtf = ((ds["compose_flops"] - ds.get("prefix_skipped_flops", 0.0)) / (ds["compose_ms"] * 1e-3) / 1e12
               if ds["compose_ms"] else 0.0)
        others["configs[2]"] = {
            "workload": "DeepSDF-style 3-(512x8)-1, linear skip over layers 1-4, seed 0, fp64, 64 dichotomy seeds; "
                        f"first {dcells} cells (max_cells cap {cap}; the full march is ~16M cells)",
            "cells": int(dcells), "waves": int(dw), "ms": d_ms, "cells_per_s": dcells / (d_ms * 1e-3),
            "compose_dmma": {"achieved_tflops": dtf, "peak_tflops": float(pk[0]),
                             "frac": dtf / pk[0] if pk[0] else None, "ms": ds["compose_ms"],
                             "share_of_march": ds["compose_ms"] / d_ms if d_ms else None},
        }
        del deng

        # configs[2] at full size: the whole ~16 M-cell march (device time, one warm-up march)
        if args.deepsdf_full:
            feng = Engine(dnet, bbox=bbox, max_cells=40_000_000)

            def frun():
                feng.reset()
                feng.seed(dseeds)
                return feng.run()
            frun()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(feng.stream)
            fw = frun()
            f1.record(feng.stream)
            torch.cuda.synchronize()
            f_ms = f0.elapsed_time(f1)
            fc = feng.counts()
            assert fc["overflow"] == 0 and not fc["capped"], "full DeepSDF march incomplete"
            fs = feng.stats()
            others["configs[2]_full"] = {
                "workload": "DeepSDF-style 3-(512x8)-1, linear skip over layers 1-4, seed 0, fp64, 64 dichotomy "
                            "seeds; the complete march (no cap)",
                "cells": int(fc["cells"]), "waves": int(fw), "ms": f_ms, "cells_per_s": fc["cells"] / (f_ms * 1e-3),
                "prefix_skipped_flops": fs["prefix_skipped_flops"],
                "timing": "CUDA events on the engine stream around reset + seed + run, after one warm-up march"}
            del feng

        # configs[4]: a batch of 64 latent-conditioned shapes (256-d code folded into the first
        # layer and skip biases of one DeepSDF decoder), one reused engine, per-shape cap
        from paper_2106_10031_b200.batch import march_batch
        lnets, _ = synth.latent_batch(n_shapes=64, latent_dim=256, width=512, depth=8, skip_at=4, seed=0)
        lcfg = marching.MarchConfig(seeds=args.seeds, rng_seed=0, bbox=bbox, max_cells=args.latent_cells)
        # warm with the same call: engine, seeding memo and the pinned host blocks of the ~1 GB of
        # per-shape results (DeepSDF keys are 512 B per cell) are then reused, as in repeated use
        march_batch(lnets, lcfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lres = march_batch(lnets, lcfg)
        torch.cuda.synchronize()
        l_s = time.perf_counter() - t0
        lcells = sum(r.report.cells_visited for _, r in lres)
        others["configs[4]"] = {
            "workload": "64 latent-conditioned shapes: 256-d code (+) xyz into a DeepSDF 3-(512x8)-1 decoder "
                        f"(code folded into first-layer / skip biases), fp64, 64 dichotomy seeds per shape, "
                        f"max_cells {args.latent_cells} per shape (the fused batch caps the total at "
                        f"{len(lnets)} x {args.latent_cells} cells)",
            "shapes": len(lres), "cells": int(lcells), "seconds": l_s, "cells_per_s": lcells / l_s,
            "per_shape_ms": 1e3 * l_s / len(lres),
            "api": "paper_2106_10031_b200.batch.march_batch(nets, MarchConfig) -> MarchResults on host; "
                   "one engine reused (am_engine_load_params), wall clock",
        }
        marching.clear_engine_cache()

    elif world > 1 and not args.no_extra:
        # the largest MLP (configs[2]) sharded over the ranks: a capped sample of its march
        from paper_2106_10031_b200 import synth
        from paper_2106_10031_b200.distributed import ShardedMarcher
        dnet = synth.deepsdf_mlp(512, 8, 4, seed=0)
        cap = args.deepsdf_cells
        dsm = ShardedMarcher(dnet, bbox=bbox, max_cells=cap)
        dseeds = dsm.sample_seeds(args.seeds, rng_seed=0)
        dsm.run(dseeds)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        rounds = dsm.run(dseeds)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        st = dsm.engine.shard_stats()
        agg = torch.tensor([(t1 - t0) * 1e3, float(st["visited"])], dtype=torch.float64, device=dev)
        dmax = agg[:1].clone()
        dist.all_reduce(dmax, op=dist.ReduceOp.MAX)
        dsum = agg[1:].clone()
        dist.all_reduce(dsum, op=dist.ReduceOp.SUM)
        d_ms, dcells = float(dmax.item()), int(dsum.item())
        others["configs[2]"] = {
            "workload": "DeepSDF-style 3-(512x8)-1, linear skip over layers 1-4, seed 0, fp64, 64 dichotomy seeds; "
                        f"first {dcells} cells (global max_cells cap {cap} shared out over {world} ranks)",
            "cells": dcells, "rounds": int(rounds), "ms": d_ms, "cells_per_s": dcells / (d_ms * 1e-3),
            "timing": "wall clock around ShardedMarcher.run, max over ranks"}
        del dsm

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = cpu_baseline_run(net, seeds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "cells_per_step": cells, "waves": int(waves),
                       "parallelism": f"dp{world} (state-hash ownership)" if world > 1 else "1 GPU",
                       "l2": "flushed between timed steps (512 MiB write)",
                       "device_march_time_s": t_step * 1e-3, "ms_steps": [round(x, 3) for x in times]},
            "roofline": roof, "kernels": kernels, "stages": stages, "cpu_baseline": cpu, "e2e": e2e,
            "other_configs": others,
            "gpu_launches": int(launches), "clocks": clocks,
            "fp64_peaks_tflops": {"dmma": float(pk[0]), "dfma": float(pk[1])},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
