#!/usr/bin/env python
"""bench.py -- SEPSO planning throughput on B200 (BASELINE.json metric: plans/sec).

Workload (N=1 headline = BASELINE config 2, the paper's dynamic scene): one
100-frame scenario stream per GPU (ScenarioConfig defaults, root seed 3 + rank,
variant sepso = evolved hypers + PI + AT, cap 30, window carryover -- the
reference's acceptance scenario, tests/acceptance.cpp:245-264).  A "step" is
one frame: plan_frame on the frozen world, then step_world.

  value  device-resident: sf_scene_batch (world, prev best, window and records
         in HBM; one fused planning launch + one on-device step_world launch
         per frame), CUDA events per step on the engine stream, L2 flushed
         between steps, max over ranks.
  e2e    the reference-facing call: sf_plan_frame with HOST world/prev/window
         buffers (one H2D + one D2H inside every step) + host step_world.

`--workload batched` runs BASELINE config 5 instead (B independent scenes per
GPU, one frame of all of them per step).  N>1 runs independent replicas (the
scene stream does not shard).  `--impl reference` times
the reference's own CPU implementation (oracle/_ref/libsfref_mt.so, compiled
unmodified from the reference headers) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

PUBLISHED_PLANS_PER_S = 1.0 / 0.0153     # C++ reference, proj/test_output.txt:28
FLOP_PER_EVAL = lambda S, E: 18 * S * E + 10 * E + 6 * S + 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sepso", choices=["sepso", "reference"])
    ap.add_argument("--workload", default="scene", choices=["scene", "batched"])
    ap.add_argument("--scenes", type=int, default=1024, help="scenes per GPU (batched)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    return ap.parse_args()


def committed_dram_bytes(kernel, grid):
    """Mean DRAM bytes (read + write) per launch of `kernel` with this grid in the
    committed ncu launch list (profiles/r01_bench_launches.csv), or None."""
    import csv
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_bench_launches.csv")
    try:
        rows = list(csv.reader(open(path)))
        hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        ix = {k: i for i, k in enumerate(rows[hdr])}
        per = {}
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[hdr + 1:]:
            if len(r) != len(rows[hdr]) or kernel not in r[ix["Kernel Name"]] or r[ix["Grid Size"]] != grid:
                continue
            if r[ix["Metric Name"]].startswith("dram__bytes_"):
                per[r[ix["ID"]]] = per.get(r[ix["ID"]], 0.0) + float(r[ix["Metric Value"]].replace(",", "")) * \
                    scale.get(r[ix["Metric Unit"]], 1.0)
        return sum(per.values()) / len(per) if per else None
    except (OSError, StopIteration, KeyError, ValueError):
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    def __init__(self, ws, rank, local, backend):
        self.ws, self.rank, self.local = ws, rank, local
        self.pg = None
        if ws > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            td.init_process_group(backend=backend, rank=rank, world_size=ws)
            self.td = td

    def barrier(self):
        if self.ws > 1:
            self.td.barrier()

    def max(self, v: float) -> float:
        if self.ws == 1:
            return v
        import torch
        dev = torch.device("cuda", self.local) if torch.cuda.is_available() else torch.device("cpu")
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.ws > 1:
            self.td.destroy_process_group()


# --------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) >= 9:
                for i, n in enumerate(names):
                    if "Active" in r[5 + i] and "Not" not in r[5 + i]:
                        reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


# ------------------------------------------------------ reference (CPU) arm
def cpu_reference_scene(frames: int, skip: int, root_seed: int = 3):
    """Reference run_scenario (unmodified, mt19937) on the host: plans/sec over
    frames [skip, frames) from the reference's own PlanRecord.wall_seconds."""
    import ctypes as C
    from oracle_lib import PlanRecord, planner_cfg, ref
    r = ref("mt")
    if r is None:
        return None
    cfg = planner_cfg(max_iters=30, window_carryover=1)
    recs = (PlanRecord * frames)()
    wall = np.zeros(frames)
    t0 = time.perf_counter()
    st = r.ref_run_scenario(root_seed, 0, frames, C.byref(cfg), recs, wall.ctypes.data_as(C.POINTER(C.c_double)))
    t1 = time.perf_counter()
    assert st == 0
    timed = wall[skip:]
    iters = np.mean([recs[i].iterations for i in range(skip, frames)])
    return {"plans_per_s": len(timed) / timed.sum(), "wall_s": t1 - t0, "mean_iterations": float(iters),
            "frames": len(timed)}


def cpu_reference_13():
    """Single-thread reference samples: one BF3 trial (G=8 N=10 T=1400, D=30) and
    one HSEF inner run (lfv_fitness, 8x170x30 on the frame-0 paper world) x 80
    candidates per evolution (hsef.hpp:125-171; the outer update is negligible)."""
    import ctypes as C
    from oracle_lib import ref, ptr, DEFAULT_GROUP_HYPERS, generate_world
    r = ref("mt")
    if r is None:
        return None
    trace, fp, ff = np.zeros(1400), np.zeros(30), C.c_double(0)
    bad = (C.c_size_t * 3)()
    t0 = time.perf_counter()
    st = r.ref_run_dtpso(3, None, 30, 30.0, 4.0, ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS)), 8, 10, 1400, 7,
                         ptr(trace), ptr(fp), C.byref(ff), bad)
    t1 = time.perf_counter()
    assert st == 0
    w = generate_world("mt", _derive(3, "world"))
    cand = np.ascontiguousarray(np.tile([1.5, 1.5, 1.5, 0.9, 0.4, 0.2], 8), dtype=np.float64)
    t2 = time.perf_counter()
    r.ref_lfv_fitness(ptr(cand), 8, 0, C.byref(w.struct()), 16, 30.0, 4.0, 8, 170, 30, 11)
    t3 = time.perf_counter()
    return {"trials_per_s": 1.0 / (t1 - t0), "ms_per_evolution": 80 * (t3 - t2) * 1e3}


def cpu_reference_batched(n_scenes: int, seconds: float = 15.0):
    """Config 5 on the host: independent cold plans (frame 0 of scenes
    0..n-1, the first frame of each scenario) on all host threads."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor
    from oracle_lib import PlanRecord, planner_cfg, ref, generate_world, oracle
    r = ref("mt")
    if r is None:
        return None
    o = oracle()
    cores = os.cpu_count() or 1
    cfg = planner_cfg(max_iters=30, window_carryover=1)

    def one(s):
        w = generate_world("mt", o.or_derive_seed(s, b"world"))
        rec = PlanRecord()
        best = np.zeros(16)
        win = np.zeros(32)
        wl = C.c_size_t(0)
        r.ref_plan_frame(C.byref(w.struct()), None, EVOLVED.ctypes.data_as(C.POINTER(C.c_double)),
                         C.byref(cfg), o.or_derive_seed_idx(s, b"plan", 0),
                         win.ctypes.data_as(C.POINTER(C.c_double)), C.byref(wl), C.byref(rec),
                         best.ctypes.data_as(C.POINTER(C.c_double)), None)
        return 1

    done = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        s = 0
        while time.perf_counter() - t0 < seconds and s < n_scenes:
            chunk = list(range(s, min(n_scenes, s + cores * 4)))
            done += sum(ex.map(one, chunk))
            s += len(chunk)
    dt = time.perf_counter() - t0
    return {"plans_per_s": done / dt, "plans": done, "cores": cores}


EVOLVED = None


def main():
    global EVOLVED
    a = parse()
    ws, rank, local = dist_env()
    if a.impl == "reference":
        return reference_arm(a, ws, rank)
    import torch
    import paper_2308_10169_b200 as pe
    EVOLVED = pe.EVOLVED_PATH_HYPERS
    torch.cuda.set_device(local)
    dist = Dist(ws, rank, local, "nccl")
    eng = pe.Engine(local, a.precision)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    root = 3 + rank
    planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    K, W = a.steps, a.warmup
    n_sc = 1 if a.workload == "scene" else a.scenes
    scen = [pe.ScenarioConfig(root_seed=(root if n_sc == 1 else rank * n_sc + s)) for s in range(n_sc)]

    # ---------------------------------------------------- device-resident value
    sb = pe.SceneBatch(eng, scen, planner, pe.EVOLVED_PATH_HYPERS, W + K)
    sb.run(W)
    eng.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = Clocks(local)
    dist.barrier()
    torch.cuda.synchronize()
    eng.synchronize()
    t_wall0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for i in range(K):
            flush.zero_()                      # L2 (126 MB) flushed between steps
            evs[i][0].record(stream)
            sb.run(1)
            evs[i][1].record(stream)
    eng.synchronize()
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    dist.barrier()
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    dev_ms = dist.max(float(np.sum(step_ms)))
    recs, _ = sb.records(W, K)
    iters = np.array([r.iterations for r in recs], dtype=np.float64)
    plans = K * n_sc
    value = plans * ws / (dev_ms / 1e3)
    evals = float(iters.sum()) * planner.groups * planner.per_group
    # kernel-only time of the fused planning kernel (same frames, timing pass)
    eng.enable_timing(True)
    sb2 = pe.SceneBatch(eng, scen, planner, pe.EVOLVED_PATH_HYPERS, W + K)
    sb2.run(W)
    eng.enable_timing(True)
    sb2.run(K)
    k_ms, k_n = eng.kernel_time()
    eng.enable_timing(False)
    recs2, _ = sb2.records(W, K)
    iters2 = np.array([r.iterations for r in recs2], dtype=np.float64)
    sb2.close()
    sb.close()
    S, E = planner.dim // 2 + 1, 32
    flop_launch = float(iters2.sum()) * planner.groups * planner.per_group * FLOP_PER_EVAL(S, E) / K
    achieved = flop_launch / (k_ms / k_n / 1e3) / 1e12
    peak = eng.measure_fp32_peak()

    # ------------------------------------------------------------ e2e (host API)
    e2e = None
    h2d = d2h = 0
    if a.workload == "scene":
        # the reference-facing loop in C++ (sf_run_scenario = run_scenario,
        # simenv.hpp:239-276): per frame sf_plan_frame with HOST world / prev /
        # window (one H2D + one D2H inside) and host step_world; per-frame wall
        # = PlanRecord.wall_seconds as the reference reports it; L2 flushed
        # between frames outside the timed calls.
        eng.set_l2_flush(256 * 1024 * 1024)
        dist.barrier()
        e_0, e_1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e_0.record(stream)
        recs_e2e = eng.run_scenario(scen[0], "sepso", W + K, planner)
        with torch.cuda.stream(stream):
            e_1.record(stream)
        torch.cuda.synchronize()
        eng.set_l2_flush(0)
        h2d, d2h = eng.last_io_bytes()
        wall = float(sum(r.wall_seconds for r in recs_e2e[W:]))
        e2e_s = dist.max(wall)
        e2e = {"value": K * ws / e2e_s, "unit": "plans/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "timing": "sum of PlanRecord.wall_seconds (host steady_clock around each sf_plan_frame call: "
                         "validate + stage + H2D copy + kernel (results stored into pinned host memory) + sync), "
                         "frames W..W+K-1",
               "whole_call_ms_events": e_0.elapsed_time(e_1),
               "mean_iterations_per_frame": float(np.mean([r.iterations for r in recs_e2e[W:]]))}
    else:
        worlds = [pe.generate_world(s, _derive(s.root_seed, "world")) for s in scen]
        seeds = [_derive(s.root_seed, "plan", 0) for s in scen]
        cfg0 = pe.PlannerConfig(max_iters_per_frame=30)
        eng.plan_frames_batched(worlds, None, None, pe.EVOLVED_PATH_HYPERS, cfg0, seeds)
        dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, min(K, 5))
        ms_tot = 0.0
        for _ in range(reps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev0.record(stream)
            eng.plan_frames_batched(worlds, None, None, pe.EVOLVED_PATH_HYPERS, cfg0, seeds)
            with torch.cuda.stream(stream):
                ev1.record(stream)
            torch.cuda.synchronize()
            ms_tot += ev0.elapsed_time(ev1)
        h2d, d2h = eng.last_io_bytes()
        e2e_ms = dist.max(ms_tot / reps)
        e2e = {"value": n_sc * ws / (e2e_ms / 1e3), "unit": "plans/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    # ------------------------------------------------------------ extra: config 5
    extra = None
    if a.workload == "scene" and not a.no_extra:
        nb = 1024
        scb = [pe.ScenarioConfig(root_seed=rank * nb + s) for s in range(nb)]
        bb = pe.SceneBatch(eng, scb, planner, pe.EVOLVED_PATH_HYPERS, 4)
        bb.run(1)
        eng.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()
            e0.record(stream)
            bb.run(3)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rb, _ = bb.records(1, 3)
        bb.close()
        extra = {"workload": f"config5: {nb} independent paper scenes per GPU, frames 1-3 (warm-started)",
                 "plans_per_s": 3 * nb * ws / (dist.max(ms) / 1e3),
                 "mean_iterations": float(np.mean([r.iterations for r in rb]))}

    # ------------------------------------------------------------ extra: Philox stream
    # the same frames with the counter-based Philox stream (north star RNG; the
    # harness build of the reference draws it): different draws, different
    # truncation points, so a different iteration count per frame
    phil = None
    if a.workload == "scene" and not a.no_extra:
        engp = pe.Engine(local, a.precision, "philox")
        sp = pe.SceneBatch(engp, scen, planner, pe.EVOLVED_PATH_HYPERS, W + K)
        sp.run(W)
        engp.synchronize()
        streamp = torch.cuda.ExternalStream(engp.stream, device=torch.device("cuda", local))
        evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        with torch.cuda.stream(streamp):
            for i in range(K):
                flush.zero_()
                evp[i][0].record(streamp)
                sp.run(1)
                evp[i][1].record(streamp)
        torch.cuda.synchronize()
        engp.synchronize()
        msp = dist.max(float(np.sum([e0.elapsed_time(e1) for e0, e1 in evp])))
        rp, _ = sp.records(W, K)
        sp.close()
        engp.close()
        phil = {"workload": "config2 frames as the headline, Philox4x32-10 counter stream",
                "plans_per_s": K * n_sc * ws / (msp / 1e3),
                "mean_iterations_per_frame": float(np.mean([r.iterations for r in rp]))}

    # ------------------------------------------------------------ extra: config 4
    # one 65,536-particle swarm (G=8 x N=8192, D=128, 1,024 obstacles), one frame
    # capped at 3 iterations: the HBM-staged path (K1 update + wide K2 fitness)
    big = None
    if a.workload == "scene" and not a.no_extra and rank == 0:
        sc4 = pe.ScenarioConfig(map_size=366.0 * np.sqrt(128.0), dynamic_obstacles=768, static_obstacles=256,
                                root_seed=1)
        w4 = pe.generate_world(sc4, 1)
        def frame4(cap, seed):
            cfg4 = pe.PlannerConfig(groups=8, per_group=8192, dim=128, max_iters_per_frame=cap, auto_truncate=False)
            eng.enable_timing(True)
            rec = eng.plan_frame(w4, None, pe.EVOLVED_PATH_HYPERS, cfg4, seed)
            ms_, _ = eng.kernel_time()
            eng.enable_timing(False)
            return ms_, rec.iterations
        frame4(1, 999)                                                      # warm-up (allocations)
        ms_a, it_a = frame4(2, 1000)
        ms_b, it_b = frame4(6, 1000)
        ms_it = (ms_b - ms_a) / max(1, it_b - it_a)       # steady iteration: K2 + K1 + bests + draws
        ms_init = ms_a - it_a * ms_it                      # init: 2RD mt19937 words (sequential) + K1 init
        S4, E4 = 65, 4 * w4.n_obstacles
        fl4 = 65536.0 * FLOP_PER_EVAL(S4, E4)
        ms4, it4 = ms_it, 1
        big = {"workload": "config4: one swarm of 65,536 particles (G=8 x N=8192), D=128, 1,024 obstacles, "
                           "cold start, iterations 3..6 vs 1..2 (HBM-staged path)",
               "ms_per_iteration": ms_it, "init_ms": ms_init, "evals_per_s": 65536.0 / (ms_it / 1e3),
               "roofline": {"kernel": "k_eval_path_wide<float> + k_step (whole iteration)", "bound": "fp32",
                            "achieved": fl4 / (ms4 / it4 / 1e3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                            "frac": fl4 / (ms4 / it4 / 1e3) / 1e12 / peak if peak else None,
                            "flop_per_eval": FLOP_PER_EVAL(S4, E4),
                            "note": "algorithmic count of SURVEY.md 8(d): every (segment, edge) pair; the map "
                                    "grid and the box cull skip most pairs, so the rate can exceed the FFMA "
                                    "peak -- kernel-quality evidence: profiles/r01_k_eval_path_wide_config4.md"}}

    # ------------------------------------------------------------ extras: configs 1 and 3
    # config 1: 1,024 BF3 (Rastrigin) trials of G=8 x N=10 x T=1400, D=30, one
    # batched launch through the public API (host buffers in and out);
    # config 3: HSEF evolutions (80 inner paper swarms x 30 iterations each) on
    # the frozen frame-0 paper world, inner (8,170,30), outer (8,10,3)
    c13 = None
    if a.workload == "scene" and not a.no_extra and rank == 0:
        seeds1 = np.arange(1, 1025, dtype=np.uint64)
        # warm-up with the same call (pinned result buffers sized once)
        eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds1)
        t0 = time.perf_counter()
        eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds1)
        t1 = time.perf_counter()
        w3 = pe.generate_world(pe.ScenarioConfig(root_seed=3), _derive(3, "world"))
        eng.evolve("path", (8, 170, 30), (8, 10, 1), 40, world=w3, dim=16)
        t2 = time.perf_counter()
        eng.evolve("path", (8, 170, 30), (8, 10, 3), 41, world=w3, dim=16)
        t3 = time.perf_counter()
        c13 = {"config1": {"workload": "1,024 BF3 trials, G=8 N=10 T=1400 D=30 (one batched call, wall)",
                           "trials_per_s": 1024 / (t1 - t0), "evals_per_s": 1024 * 80 * 1400 / (t1 - t0)},
               "config3": {"workload": "HSEF evolve, inner (8,170,30) path on the frame-0 paper world, outer (8,10,3)",
                           "ms_per_evolution": (t3 - t2) / 3 * 1e3,
                           "inner_evals_per_s": 3 * 80 * 1360 * 30 / (t3 - t2)}}
        ref13 = cpu_reference_13() if not a.no_cpu_baseline else None
        if ref13:
            c13["config1"]["reference_1thread_trials_per_s"] = ref13["trials_per_s"]
            c13["config3"]["reference_1thread_ms_per_evolution"] = ref13["ms_per_evolution"]

    # ------------------------------------------------------------ CPU baseline
    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        if a.workload == "scene":
            c = cpu_reference_scene(100, 0)
            if c:
                cpu = {"value": c["plans_per_s"], "unit": "plans/s", "cores": 1, "kind": "reference",
                       "sample": f"reference run_scenario (unmodified, mt19937), root seed 3, 100 frames, "
                                 f"cap 30, carryover; mean {c['mean_iterations']:.1f} iterations/frame"}
        else:
            c = cpu_reference_batched(min(n_sc, 4096))
            if c:
                cpu = {"value": c["plans_per_s"], "unit": "plans/s", "cores": c["cores"], "kind": "reference",
                       "sample": f"{c['plans']} cold plans (frame 0 of scenes 0..), scene-parallel, ~15 s"}

    if rank == 0:
        cpu_thr = os.cpu_count() or 1
        line = {
            "metric": "plans_per_sec",
            "value": value,
            "unit": "plans/s",
            "n_gpus": ws,
            "steps": K,
            "warmup": W,
            "ms_per_step": dev_ms / K,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": value / PUBLISHED_PLANS_PER_S if a.workload == "scene" else None,
            "dtype": a.precision,
            "data": "synthetic (seeded generate_world scenes; the reference's mt19937_64 draw stream, generated on the device)",
            "config": {
                "workload": ("config2: paper dynamic scene (366 cm, 6 dynamic + 2 static obstacles), "
                             "SEPSO evolved hypers + PI + AT, G=8 N=170 D=16, cap 30, window carryover, "
                             f"root seed {root}; one frame per step" if a.workload == "scene" else
                             f"config5: {n_sc} independent paper scenes per GPU, one frame each per step"),
                "scenes_per_gpu": n_sc,
                "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                "l2": "flushed between steps (256 MiB write)",
                "mean_iterations_per_frame": float(iters.mean()),
                "fitness_evals": evals,
                "evals_per_sec": evals * ws / (dev_ms / 1e3),
            },
            "roofline": {
                "kernel": "swarm_kernel<float,path> (fused frame: fitness+bests+AT+update)",
                "bound": "fp32",
                "achieved": achieved,
                "peak": peak,
                "peak_source": "measured FFMA probe (sf_measure_fp32_peak) on this GPU",
                "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None,
                "traffic": committed_dram_bytes("swarm_kernel<float, 1, 0>", "(16, 1, 1)"),
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel, "
                                  "profiles/r01_bench_launches.csv (ncu launch list of this bench, cold-cache replays)",
                "flop_per_launch": flop_launch,
                "flop_per_eval": FLOP_PER_EVAL(S, E),
                "avg_launch_us": 1e3 * k_ms / k_n,
                "launches": int(k_n),
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": K,                        # one fused launch per frame (world step included)
            "clocks": clk,
            "batched": extra,
            "config4": big,
            "philox": phil,
            "configs_1_3": c13,
            "host_threads": cpu_thr,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    dist.close()


def _derive(root, tag, idx=None):
    from oracle_lib import oracle   # seed derivation only (rng.hpp:52-59)
    o = oracle()
    return o.or_derive_seed(root, tag.encode()) if idx is None else o.or_derive_seed_idx(root, tag.encode(), idx)


def reference_arm(a, ws, rank):
    if rank != 0:
        return 0
    from oracle_lib import ref
    if ref("mt") is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsfref_mt.so not built"}))
        return 0
    K, W = a.steps, a.warmup
    if a.workload == "scene":
        c = cpu_reference_scene(W + K, W)
        value, cores = c["plans_per_s"], 1
        sample = f"reference run_scenario root seed 3, frames {W}..{W + K - 1} timed (cap 30, carryover)"
        cfgd = {"workload": "config2: paper dynamic scene, reference CPU (unmodified, mt19937)",
                "mean_iterations_per_frame": c["mean_iterations"]}
    else:
        global EVOLVED
        from oracle_lib import EVOLVED_PATH_HYPERS
        EVOLVED = np.ascontiguousarray(EVOLVED_PATH_HYPERS)
        c = cpu_reference_batched(a.scenes * max(1, a.gpus), seconds=20.0)
        value, cores = c["plans_per_s"], c["cores"]
        sample = f"{c['plans']} cold plans, scene-parallel on {cores} threads"
        cfgd = {"workload": "config5: independent paper scenes, reference CPU"}
    line = {"impl": "reference", "metric": "plans_per_sec", "value": value, "unit": "plans/s",
            "n_gpus": a.gpus, "steps": K, "warmup": W, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": value / PUBLISHED_PLANS_PER_S,
            "dtype": "fp64", "data": "synthetic", "config": cfgd,
            "cpu_baseline": {"value": value, "unit": "plans/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
