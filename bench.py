#!/usr/bin/env python
"""Benchmark: FMM DDM matvec on config 5 (N = 1e6 elastic elements, leaf 64,
p = 20) — BASELINE.json metric "FMM DDM matvec interactions/s and GMRES solve
time (fp64) vs roofline, 1/2/4/8 GPU".

A step is one FMM matvec y = A D (prep, P2M, M2M, M2L, L2L, P2P, L2P+finalize;
the tree is built once per geometry, and timed separately).
value = dense-equivalent interactions/s = N^2 per matvec (whole job).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: launched by torchrun, one rank per GPU, NCCL)
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

METRIC = ("FMM DDM matvec interactions/s and GMRES solve time (fp64) vs roofline, "
          "1/2/4/8 GPU")
UNIT = "interactions/s"
FLOP_PER_PAIR = 45          # P2P algorithmic unit, fixed since round 1: the record update as first written (16 FMA + 5 MUL + 8 ADD, cubic reciprocal refinement); the round-2 kernel executes 43 (K-form record, one-step reciprocal)
FP64_INSTR_PER_PAIR = 25    # fp64-pipe instructions per record and target in the SASS of p2p_leaf_kernel's loop (21 DFMA + 2 DADD + 2 DMUL, + 1 MUFU.RCP64H; 28 in round 1)
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, local, world


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile(prefix="clocks", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
        loaded = [v for v in sm if v > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def _host_info() -> dict:
    info = {"nproc": os.cpu_count()}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


def _oracle_rows(args):
    from oracle import elastic as OE
    g, G, nu, Dv, idx = args
    return OE.matvec_rows(g, G, nu, Dv, idx)


def cpu_baseline_oracle(g, mat, Dv, rows: int, workers: int | None = None):
    """The oracle (numpy, fp64, as it stands) on a bounded sample: `rows` target
    rows of config 5 against all N sources (oracle/elastic.matvec_rows), the
    rows split over `workers` processes (default: every host core).  Returns
    (interactions/s, seconds, workers)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    workers = workers or os.cpu_count() or 1
    idx = np.random.default_rng(1234).choice(g.n, rows, replace=False)
    chunks = [c for c in np.array_split(idx, workers) if c.size]
    jobs = [(g, mat["G"], mat["nu"], Dv, c) for c in chunks]
    with ProcessPoolExecutor(max_workers=len(jobs), mp_context=mp.get_context("spawn")) as ex:
        list(ex.map(_oracle_rows, jobs[:1]))        # worker start-up outside the timing
        t0 = time.perf_counter()
        list(ex.map(_oracle_rows, jobs))
        dt = time.perf_counter() - t0
    return rows * g.n / dt, dt, len(jobs)


def oracle_gmres_cfg2():
    """The oracle's dense GMRES on config 2 (oracle/gmres.py: CGS2, Givens,
    unpreconditioned, tol 1e-10) beside the GPU solve: assembly and solve
    times, iterations; numpy BLAS threads as configured on the host."""
    from oracle import elastic as OE
    from oracle import gmres as OG
    from synth import CONFIGS, make_config
    c = CONFIGS[2]
    g = make_config(2)
    t0 = time.perf_counter()
    A = OE.assemble_dense(g, c["material"]["G"], c["material"]["nu"])
    t1 = time.perf_counter()
    b = OE.farfield_rhs(g, c["load"]).reshape(-1)
    x, it, rr, ok = OG.gmres(lambda v: A @ v, b, tol=c["tol"], restart=2000, max_iter=10000)
    t2 = time.perf_counter()
    try:
        from threadpoolctl import threadpool_info
        threads = max((d.get("num_threads", 1) for d in threadpool_info()), default=1)
    except Exception:
        threads = None
    return {"assembly_s": t1 - t0, "solve_s": t2 - t1, "iters": it, "rel_resid": rr,
            "blas_threads": threads, "precond": "none (the oracle follows the paper's plain GMRES)"}


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, rank 0 only."""
    rank, _, world = _dist()
    if rank != 0:
        return
    from synth import CONFIGS, make_config, random_dd
    c = CONFIGS[args.config]
    g = make_config(args.config)
    Dv = random_dd(g.n, 2, c["d_seed"])
    rows = args.ref_rows
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_baseline_oracle(g, c["material"], Dv, max(cores, rows // 4))
    times = []
    for _ in range(args.steps):
        v, dt, cores = cpu_baseline_oracle(g, c["material"], Dv, rows)
        times.append(dt)
    tot = sum(times)
    value = args.steps * rows * g.n / tot
    sample = (f"{rows} seeded target rows x all {g.n} sources per step, split over {cores} "
              f"processes (oracle.elastic.matvec_rows, numpy fp64)")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": c["name"], "N": g.n, "leaf": c["leaf"], "p": c["p"]},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": sample, "host": _host_info()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1812_05087_b200 as D
    from synth import CONFIGS, make_config, random_dd

    rank, local, world = _dist()
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [D.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = D.Context(local, rank, world, uid)
    c = CONFIGS[args.config]
    p = args.p or c["p"]
    g = make_config(args.config)
    n = g.n
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    xc, yc, hl, be = f(g.xc), f(g.yc), f(g.half_len), f(g.beta)
    mat = D.material_from_dict(c["material"])
    stream = torch.cuda.current_stream()

    # tree (built once per geometry): the first build in the
    # process includes one-time kernel-module loading; the tree used below is
    # the second build (steady state), timed per stage by the library
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = D.Tree(ctx, xc, yc, hl, be, leaf_size=c["leaf"], order_p=p)
    torch.cuda.synchronize()
    tree_first_ms = (time.perf_counter() - t0) * 1e3
    tree.free()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = D.Tree(ctx, xc, yc, hl, be, leaf_size=c["leaf"], order_p=p)
    torch.cuda.synchronize()
    tree_ms = (time.perf_counter() - t0) * 1e3
    tree_stages = tree.build_times()
    cnt = tree.counts

    Dv_host = random_dd(n, 2, c["d_seed"])
    Dd = f(Dv_host)
    y = torch.empty_like(Dd)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    for _ in range(args.warmup):
        D.matvec(ctx, tree, mat, Dd, y)
    torch.cuda.synchronize()

    # ---- timed region: K matvecs, L2 flushed between steps (outside the events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    for k in range(args.steps):
        flush.zero_()
        starts[k].record()
        D.matvec(ctx, tree, mat, Dd, y)
        ends[k].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = args.steps * float(n) * float(n) / (tot_ms * 1e-3)

    # ---- end to end through the public API: every step copies its D from
    # pinned host memory, runs the matvec and copies y back to pinned host
    # memory.  Steps are pipelined over two device buffer pairs: the H2D of
    # step k+1 (copy stream) and the D2H of step k-1 (second copy stream)
    # overlap the matvec of step k (compute stream); events order the reuse.
    hD = torch.from_numpy(Dv_host).pin_memory()
    hy = [torch.empty_like(hD).pin_memory() for _ in range(2)]
    dD = [torch.empty_like(Dd) for _ in range(2)]
    dy = [torch.empty_like(Dd) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    comp = torch.cuda.current_stream()

    def e2e_steps(k_steps):
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_mv = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        for k in range(k_steps):
            b = k & 1
            with torch.cuda.stream(s_in):
                if used[b]:
                    s_in.wait_event(ev_mv[b])          # matvec k-2 done reading dD[b]
                dD[b].copy_(hD, non_blocking=True)
                ev_in[b].record(s_in)
            comp.wait_event(ev_in[b])
            if used[b]:
                comp.wait_event(ev_out[b])             # D2H of step k-2 done with dy[b]
            D.matvec(ctx, tree, mat, dD[b], dy[b], stream=comp)
            ev_mv[b].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_mv[b])
                hy[b].copy_(dy[b], non_blocking=True)
                ev_out[b].record(s_out)
            used[b] = True

    e2e_steps(4)   # warm-up (graph capture of both buffer pairs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(s_in)
    e2e_steps(args.steps)
    ee1.record(s_out)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = args.steps * float(n) * float(n) / (e2e_ms * 1e-3)
    y_e2e_ok = bool(torch.equal(hy[(args.steps - 1) & 1].to(dev), y)) if world == 1 else None

    # ---- per-stage CUDA events (separate instrumented run) for the roofline
    # serial schedule: every stage's events bracket that stage's kernels alone
    # (in the timed step the near field overlaps the far-field chain)
    ctx.set_profiling(True, serial=True)
    stages = {k: 0.0 for k in ("prep", "p2m", "m2m", "m2l", "l2l", "l2p", "p2p", "final", "comm",
                               "p2l")}
    nprof = max(3, min(args.steps, 10))
    for _ in range(nprof):
        flush.zero_()
        D.matvec(ctx, tree, mat, Dd, y)
        torch.cuda.synchronize()
        for k, v in ctx.stage_times().items():
            stages[k] += v / nprof
    # the same events on the normal (concurrent) schedule: the near field's
    # span while it shares the GPU with the far-field chain
    ctx.set_profiling(True, serial=False)
    p2p_conc = 0.0
    for _ in range(nprof):
        flush.zero_()
        D.matvec(ctx, tree, mat, Dd, y)
        torch.cuda.synchronize()
        p2p_conc += ctx.stage_times()["p2p"] / nprof
    ctx.set_profiling(False)
    fp64_peak = ctx_probe_fp64(ctx)
    kern = kernel_rooflines(tree, cnt, stages, tree_stages, p, fp64_peak, world)
    owned_pairs = cnt["NEAR_PAIRS_P2P"] / world   # approx. per rank for N > 1 (U minus X)
    p2p_ms = stages["p2p"]
    achieved = owned_pairs * FLOP_PER_PAIR / (p2p_ms * 1e-3) / 1e12
    levels = cnt["LEVELS"]
    # per matvec: prep_sources, p2p_kernel, p2m_kernel, m2m_level_kernel per
    # level 2..L-2 with parents, m2l_kernel, l2l_level_kernel per level 3..L-1,
    # l2p_kernel, finalize_kernel = 2 L for L levels (24 at L = 12; the list in
    # profiles/r1_launches_cfg5_summary.txt), replayed as one CUDA graph
    # (+ unpack_allgather and scatter_user when the rows are exchanged)
    launches_per_step = 2 * levels
    if world > 1:
        launches_per_step += 2

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": c["name"], "N": n, "leaf": c["leaf"], "p": p,
                      "elements_per_fracture": 100, "fractures": 10000, "box_m": 2000,
                      "parallelism": f"morton-leaf-partition x{world}",
                      "l2": "flushed between steps (256 MiB write, outside the step events)",
                      "tree_build_ms": tree_ms, "tree_build_first_ms": tree_first_ms,
                      "tree_build_stage_ms": tree_stages,
                      "cells": cnt["CELLS"], "leaves": cnt["LEAVES"],
                      "levels": levels, "v_pairs": cnt["V"], "near_pairs": cnt["NEAR_PAIRS"]},
           "stage_ms": stages,
           "kernels": kern,
           "roofline": {"bound": "alu", "kernel": "p2p_leaf_kernel (fp64 pipe)",
                        "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                        "frac": achieved / fp64_peak if fp64_peak else None,
                        "traffic": _ncu_traffic("p2p_leaf_kernel"),
                        "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one "
                                          "ncu --set full capture (profiles/ncu_traffic.json)",
                        "traffic_note": "algorithmic: 96-B source records once (~100 MB) + "
                                        "targets (~48 MB); leaf CTAs launched heaviest-first "
                                        "re-read shared U-list records from DRAM (~264 MB; "
                                        "Morton order, DDM_P2P_ORDER=0, reads about the "
                                        "algorithmic bytes at a 1.2 % slower step): the kernel "
                                        "is fp64-bound, ~0.45 TB/s of DRAM",
                        "peak_source": "measured DFMA-chain probe (ddm_probe_fp64) on this GPU",
                        "flop_per_pair": FLOP_PER_PAIR,
                        "fp64_pipe_frac": (owned_pairs * FP64_INSTR_PER_PAIR / (p2p_ms * 1e-3)
                                           / (fp64_peak * 1e12 / 2.0)) if fp64_peak else None,
                        "fp64_pipe_frac_note": "fp64-pipe instructions issued / peak instruction "
                                               "rate (peak TFLOP/s / 2 flop per DFMA)",
                        "kernel_ms": p2p_ms,
                        "kernel_ms_source": "CUDA events on the launching stream, serial "
                                            "instrumented matvecs after the timed region",
                        "p2p_share_of_serial_step": p2p_ms / sum(stages.values()),
                        "kernel_ms_concurrent": p2p_conc,
                        "kernel_ms_concurrent_note": "P2P span on its own stream in the "
                                                     "concurrent schedule (shares the SMs with "
                                                     "the far-field chain)"},
           "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(hD.numel() * 8),
                   "d2h_bytes_per_step": int(hy[0].numel() * 8),
                   "ms_per_step": e2e_ms / args.steps,
                   "pipelined": "H2D of step k+1 and D2H of step k-1 overlap matvec k "
                                "(two buffer pairs, two copy streams)",
                   "result_matches_device_run": y_e2e_ok},
           "gpu_launches": launches_per_step * args.steps,
           "clocks": clocks}

    if rank == 0 and world == 1 and not args.no_extras:
        # the paper's own far field (Chebyshev bbFMM, NCheb3 / NCheb6) on the
        # same tree and input
        out["bbfmm"] = bbfmm_extra(D, ctx, torch, tree, mat, Dd, y, flush, cnt, fp64_peak)
        # GMRES solve time on config 2 (the metric's second half), at p and p*
        out["gmres"] = gmres_extra(D, ctx, torch, dev, args.march_steps)
        gv, gdt, gw = cpu_baseline_oracle(g, c["material"], Dv_host, args.cpu_rows)
        out["cpu_baseline"] = {"value": gv, "unit": UNIT, "cores": gw, "kind": "oracle",
                               "sample": f"{args.cpu_rows} seeded target rows x all {n} sources, "
                                         f"split over {gw} processes (oracle.elastic.matvec_rows, "
                                         f"numpy fp64, {gdt:.1f} s)",
                               "host": _host_info(),
                               "gmres_cfg2": oracle_gmres_cfg2()}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


HBM_PEAK_FALLBACK = 6650.0   # GB/s, the fallback B200_PROFILING.md states when MEASURED_PEAKS.json is absent


def _hbm_peak() -> tuple:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy)"
    except Exception:
        return HBM_PEAK_FALLBACK, "of fallback: 6650 GB/s (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


def kernel_rooflines(tree, cnt, stages, tree_stages, p, fp64_peak, world):
    """Roofline fraction of every stage of the step (serial instrumented
    matvecs, CUDA events on the launching stream) and of the tree build
    stages, in SURVEY.md §8(d).2 work units (DESIGN.md §7.1 states each unit
    and where the implementation executes a different amount of work):
      fp64 stages: algorithmic flop / time / measured fp64 peak (DFMA probe);
      HBM stages : algorithmic bytes / time / measured HBM copy bandwidth."""
    n = cnt["N"]
    lev = tree.export("LEVEL")
    leaves = tree.export("LEAVES")
    count = tree.export("COUNT")
    woff = tree.export("W_OFF")
    n_l3 = int((lev >= 3).sum())                 # cells with a parent of level >= 2
    el_w = int((count[leaves] * np.diff(woff)).sum())   # (element, W cell) pairs
    T = 12800                                      # flop per translation: dense 80 x 80 real operator
    hbm, hbm_src = _hbm_peak()
    depth = cnt["LEVELS"] - 1
    sort_passes = max(1, -(-2 * depth // 8))
    rows = {
        "prep": ("hbm", 165.0 * n, "B", "165 B/elem: D (16, gathered through perm), geometry "
                 "(40), stream tables (13) in; 80-B near-field record and D sorted (16) out"),
        "p2m": ("fp64", 40.0 * p * n, "flop", "SURVEY 40 p flop/elem (exact segment moments)"),
        "m2m": ("fp64", float(T) * n_l3, "flop", "SURVEY 12 800 flop per child translation "
                "(executed: separable Pascal form, about half)"),
        "m2l": ("fp64", float(T) * cnt["V"], "flop", "SURVEY 12 800 flop per V pair (executed on "
                "DMMA: 9 x DMMA.8x8x4 = 4 608 flop per pair, Pascal form)"),
        "l2l": ("fp64", float(T) * n_l3, "flop", "SURVEY 12 800 flop per parent-to-child "
                "translation"),
        "l2p": ("fp64", (24.0 * p + 20) * n + (24.0 * p + 30) * el_w, "flop",
                f"(24 p + 20) flop/elem local + (24 p + 30) per (element, W cell) M2P pair "
                f"({el_w} pairs)"),
        "p2p": ("fp64", FLOP_PER_PAIR * cnt["NEAR_PAIRS_P2P"] / world, "flop",
                "45 flop per near pair (the round-1 node-sharing record update as written; "
                "the round-2 kernel executes 43 with 25 fp64 instructions, DESIGN.md §4.2c)"),
        "final": ("hbm", 52.0 * n, "B", "52 B/elem: near (16) + far (16) + perm (4) in, y (16) out"),
    }
    out = {}
    for k, (bound, work, unit, note) in rows.items():
        ms = stages.get(k, 0.0)
        if ms <= 0:
            continue
        if bound == "fp64":
            ach = work / (ms * 1e-3) / 1e12
            out[k] = {"bound": "alu", "unit": "TFLOP/s", "achieved": ach, "peak": fp64_peak,
                      "frac": ach / fp64_peak if fp64_peak else None, "kernel_ms": ms,
                      "work": work, "work_unit": unit, "note": note}
        else:
            ach = work / (ms * 1e-3) / 1e9
            out[k] = {"bound": "hbm", "unit": "GB/s", "achieved": ach, "peak": hbm,
                      "frac": ach / hbm, "kernel_ms": ms, "work": work, "work_unit": unit,
                      "note": note}
    m2l_exec = 4608.0 * cnt["V"] / (stages["m2l"] * 1e-3) / 1e12 if stages.get("m2l") else None
    if m2l_exec and "m2l" in out:
        out["m2l"]["executed_dmma_tflops"] = m2l_exec
        out["m2l"]["executed_dmma_frac"] = m2l_exec / fp64_peak if fp64_peak else None
    tb = {
        "keys": (28.0 * n, "SURVEY 28 B/elem (centres in, key + index out)"),
        "sort": ((24.0 * sort_passes + 8.0) * n, f"SURVEY {sort_passes} passes x 24 B/elem + 8 "
                 "B/elem histogram (executed: 8 passes of 8-bit digits over the 60-bit key, "
                 "for the bit-exact full-key order)"),
        "cells": (24.0 * n * depth, "24 B/elem per level"),
        "lists": (48.0 * cnt["CELLS"] + 4.0 * (cnt["V"] + 2 * cnt["URANGES"] + cnt["W"]),
                  "48 B/cell + 4 B per V, U-range bound and W entry"),
    }
    tree_out = {}
    for k, (byt, note) in tb.items():
        ms = tree_stages.get(k, 0.0)
        if ms > 0:
            ach = byt / (ms * 1e-3) / 1e9
            tree_out[k] = {"bound": "hbm", "unit": "GB/s", "achieved": ach, "peak": hbm,
                           "frac": ach / hbm, "kernel_ms": ms, "work": byt, "work_unit": "B",
                           "note": note + " (stage span incl. host gaps)"}
    return {"step": out, "tree_build": tree_out, "fp64_peak_source":
            "measured DFMA-chain probe (ddm_probe_fp64) on this GPU", "hbm_peak_source": hbm_src,
            "time_source": "CUDA events around each stage's kernels, serial schedule, after the "
                           "timed region (profiles/r2_step_ncu_summary.txt has the ncu rows)"}


def _ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)[kernel]["dram_bytes"]
    except Exception:
        return None


def ctx_probe_fp64(ctx) -> float:
    import ctypes as C
    from paper_1812_05087_b200 import _lib as L
    import torch
    v = C.c_double(0.0)
    rc = L.lib.ddm_probe_fp64(ctx._h, C.byref(v), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    return v.value if rc == 0 else None


def _poro_rc(c, g, tau):
    """sqrt(160 c tau) + 2 max(a): the min leaf side for the poroelastic far field."""
    m = c["material"]
    G, nu, nuu, al, kap = m["G"], m["nu"], m["nu_u"], m["alpha"], m["kappa"]
    M = 2 * G * (nuu - nu) / (al * al * (1 - 2 * nuu) * (1 - 2 * nu))
    S = al * al * (1 - 2 * nu) / (2 * G * (1 - nu)) + 1 / M
    return (160 * (kap / S) * tau) ** 0.5 + 2 * float(g.half_len.max())


# fp64-pipe instructions per node pair of bb_m2l_kernel<6> (DFMA + DMUL + DADD
# of the fully unrolled node loop / 36, cuobjdump -sass)
BB_M2L_INSTR_PER_NODE_PAIR = 33


def bbfmm_extra(D, ctx, torch, tree, mat, Dd, y, flush, cnt, fp64_peak, reps: int = 20):
    """Matvec time of the bbFMM far field at n = 3 and 6 (the paper's NCheb3 /
    NCheb6) on the bench workload: CUDA events around `reps`
    matvecs (L2 flushed before each, outside the events), serial per-stage
    times, the relative L2 difference from the p = 20 series matvec (whose own
    error is ~1e-10), and the fp64-pipe fraction of the dominant kernel (M2L)."""
    ref = torch.empty_like(Dd)
    D.matvec(ctx, tree, mat, Dd, ref)
    res = {}
    for n in (3, 6):
        mode = f"bbfmm{n}"
        for _ in range(3):
            D.matvec(ctx, tree, mat, Dd, y, mode=mode)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            D.matvec(ctx, tree, mat, Dd, y, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        err = (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()
        ctx.set_profiling(True, serial=True)
        st = {}
        for _ in range(3):
            flush.zero_()
            D.matvec(ctx, tree, mat, Dd, y, mode=mode)
            torch.cuda.synchronize()
            for k, v in ctx.stage_times().items():
                st[k] = st.get(k, 0.0) + v / 3
        ctx.set_profiling(False)
        node_pairs = cnt["V"] * (n * n) ** 2
        r = {"ms_per_matvec": tot / reps, "rel_diff_vs_series_p20": err,
             "serial_stage_ms": {k: v for k, v in st.items() if v > 0},
             "m2l_node_pairs": node_pairs}
        if n == 6 and fp64_peak and st.get("m2l"):
            r["m2l_fp64_pipe_frac"] = (node_pairs * BB_M2L_INSTR_PER_NODE_PAIR
                                       / (st["m2l"] * 1e-3) / (fp64_peak * 1e12 / 2.0))
        res[mode] = r
    return res


def gmres_extra(D, ctx, torch, dev, march_steps: int):
    """The metric's second half: GMRES solve times (device-synchronised wall
    clock around ddm_gmres_solve) on config 2 (elastic, p and p*) and config 3
    (poroelastic, full size), poroelastic matvec times, and config 4 time
    marching (history + GMRES per step) over `march_steps` steps (all 200 by
    default), with the history sum timed in the fast form and per lag at the
    last step."""
    from synth import CONFIGS, make_config
    res = {}
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)

    def timed(fn, reps=1):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3, r

    def steady_mv(fn):
        # the first poroelastic matvec on the fresh tree (one-time workspace
        # allocation, source stream build, first-use module loading, near
        # field on the fly), then the second (builds the near-field cache);
        # matvec_ms below is the steady state (cached blocks, graph replay)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        first = (time.perf_counter() - t0) * 1e3
        fn()
        torch.cuda.synchronize()
        return first

    g = make_config(2)
    c = CONFIGS[2]
    mat = D.material_from_dict(c["material"])
    for p in (c["p"], c["p_star"]):
        tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                      order_p=p)
        ld = c["load"]
        b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
        ms, (x, it, rr) = timed(lambda: D.gmres_solve(ctx, tree, mat, b, tol=c["tol"]))
        res[f"cfg2_p{p}"] = {"solve_ms": ms, "iters": it, "rel_resid": rr}
        tree.free()
    # config 3: poroelastic, N = 20000 (60000 unknowns), one temporal element
    g = make_config(3)
    c = CONFIGS[3]
    mat = D.material_from_dict(c["material"])
    tau = c["dt"]
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                  order_p=c["p_star"], min_leaf_side=_poro_rc(c, g, tau))
    ld = c["load"]
    b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=True,
                       b_p=ld["sh"] + ld["p_f"] - ld["p0"])
    y = torch.empty_like(b)
    first_ms = steady_mv(lambda: D.matvec(ctx, tree, mat, b, y, elapsed=tau))
    mv_ms, _ = timed(lambda: D.matvec(ctx, tree, mat, b, y, elapsed=tau), reps=20)
    ms, (x, it, rr) = timed(lambda: D.gmres_solve(ctx, tree, mat, b, dt=tau, tol=c["tol"],
                                                   restart=3000, max_iter=6000))
    res["cfg3_poro"] = {"solve_ms": ms, "iters": it, "rel_resid": rr, "matvec_ms": mv_ms,
                        "matvec_first_ms": first_ms,
                        "p": c["p_star"], "near_pairs": tree.counts["NEAR_PAIRS"]}
    # CGS2 roofline (SURVEY 8(d).2 unit, DESIGN 4.1 a12): Arnoldi step k reads the
    # k+1 basis vectors four times (dot + axpy, two passes) = 4 (k+1) dof 8 B.  The
    # time is everything in the solve that is not a matvec (CGS2, preconditioner,
    # Givens, residual read-backs), so the fraction is a lower bound for the passes.
    dof = int(b.numel())
    cgs_bytes = 32.0 * dof * it * (it + 1) / 2
    rest_ms = max(ms - it * mv_ms, 1e-9)
    hbm, hbm_src = _hbm_peak()
    res["cfg3_poro"]["cgs2"] = {
        "bound": "hbm", "unit": "GB/s", "achieved": cgs_bytes / (rest_ms * 1e-3) / 1e9,
        "peak": hbm, "frac": cgs_bytes / (rest_ms * 1e-3) / 1e9 / hbm,
        "bytes_per_iter_mean": cgs_bytes / max(it, 1), "non_matvec_ms_per_iter": rest_ms / max(it, 1),
        "peak_source": hbm_src,
        "note": "time = solve - iters x steady matvec (CGS2 + preconditioner + Givens + "
                "read-backs); the basis (iters x dof x 8 B) stays in the 126 MB L2, the HBM "
                "copy peak is the conservative denominator"}
    tree.free()
    # config 4: poroelastic time marching (first march_steps of the 200 steps)
    g = make_config(4)
    c = CONFIGS[4]
    mat = D.material_from_dict(c["material"])
    dt = c["dt"]
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                  order_p=c["p_star"], min_leaf_side=_poro_rc(c, g, (c["steps"] + 1) * dt))
    ld = c["load"]
    b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False,
                       b_p=ld["p_f"] - ld["p0"])
    y = torch.empty_like(b)
    first4 = steady_mv(lambda: D.matvec(ctx, tree, mat, b, y, elapsed=dt))
    mv_ms, _ = timed(lambda: D.matvec(ctx, tree, mat, b, y, elapsed=dt), reps=20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Dh, st = D.march(ctx, tree, mat, dt, b, march_steps, tol=c["tol"])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    # the history / GMRES split: a second march with per-step synchronised timers
    _, st = D.march(ctx, tree, mat, dt, b, march_steps, tol=c["tol"], timing=True)
    h = march_steps - 1
    hf, _ = timed(lambda: D.history_apply(ctx, tree, mat, dt, Dh[:h], mode="fmm"))
    hp, _ = timed(lambda: D.history_apply(ctx, tree, mat, dt, Dh[:h], mode="perlag"))
    its = [s["iters"] for s in st]
    res["cfg4_march"] = {"steps": march_steps, "of_steps": c["steps"], "wall_s": wall,
                         "gmres_iters": {"first": its[0], "min": min(its), "max": max(its),
                                         "mean": sum(its) / len(its), "total": sum(its)},
                         "max_rel_resid": max(s["rel_resid"] for s in st),
                         "gmres_s": sum(s["gmres_s"] for s in st),
                         "history_s": sum(s["history_s"] for s in st), "matvec_ms": mv_ms,
                         "matvec_first_ms": first4,
                         f"history_fast_h{h}_ms": hf, f"history_perlag_h{h}_ms": hp}
    tree.free()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--march-steps", type=int, default=200)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
