#!/usr/bin/env python
"""bench.py -- SEPSO planning throughput on B200 (BASELINE.json metric: plans/sec).

Headline (N=1) = BASELINE config 2, the paper's dynamic scene: the reference's
acceptance scenario (ScenarioConfig defaults, root seed 3 + rank, variant sepso
= evolved hypers + PI + AT, cap 30, window carryover; acceptance.cpp:245-264),
frames W..W+K-1 timed.  A "step" is one frame: plan_frame on the frozen world,
then step_world.

  value  device-resident: sf_scene_batch (world, prev best, window and records
         in HBM; one fused launch per frame that plans and steps the world),
         CUDA events per step on the engine stream, L2 flushed between steps,
         max over ranks.
  e2e    the reference-facing call: sf_run_scenario = per frame sf_plan_frame
         with HOST world / prev / window buffers (inputs in, record out inside
         the call) + host step_world; wall = PlanRecord.wall_seconds.

Extras, each with its own roofline and an all-cores CPU baseline of the
unmodified reference (oracle/_ref) timed in the same run: config 5 (batched
scenes, sharded over ranks), config 4 (one 65,536-particle swarm; K1 and K2),
config 3 (HSEF evolution, candidates sharded over ranks), config 1 (benchmark
trials, sharded over ranks), the FP64 parity engine on the headline frames,
and the Philox stream.  N>1 runs the headline as independent replicas (the
scene stream does not shard).  `--impl reference` times
the reference's own CPU implementation on the headline workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

FLOP_PER_EVAL = lambda S, E: 18 * S * E + 10 * E + 6 * S + 3
# the headline workload, word for word the same in both arms
WORKLOAD_C2 = ("config2: paper dynamic scene (366 cm, 6 dynamic + 2 static obstacles), SEPSO evolved hypers "
               "+ PI + AT, G=8 N=170 D=16, cap 30, window carryover, root seed 3 (+rank); frames W..W+K-1, "
               "one frame per step")
PROFILE_CSV = "profiles/r02_bench_launches.csv"        # ncu launch list of this bench (roofline.traffic)
LATENCY_KERNEL = "swarm_kernel<float, 1, 0, 896, 0, 1>"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sepso", choices=["sepso", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0, help="bound of each all-cores CPU baseline")
    return ap.parse_args()


def committed_dram_bytes(kernel, grid, path=PROFILE_CSV):
    """Mean DRAM bytes (read + write) per launch of `kernel` with this grid in a
    committed ncu launch list, or None."""
    import csv
    try:
        rows = list(csv.reader(open(os.path.join(ROOT, path))))
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


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


class Dist:
    def __init__(self, ws, rank, local, backend):
        self.ws, self.rank, self.local = ws, rank, local
        if ws > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            td.init_process_group(backend=backend, rank=rank, world_size=ws)
            self.td = td

    def barrier(self):
        if self.ws > 1:
            self.td.barrier()

    def _t(self, a):
        import torch
        dev = torch.device("cuda", self.local) if torch.cuda.is_available() else torch.device("cpu")
        return torch.tensor(a, dtype=torch.float64, device=dev)

    def max(self, v: float) -> float:
        if self.ws == 1:
            return v
        t = self._t([v])
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if self.ws == 1:
            return v
        t = self._t([v])
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())

    def allgather_bytes(self, send: bytes) -> bytes:
        """all ranks' equal-size byte strings, rank order (host exchange for the engine)."""
        if self.ws == 1:
            return send
        import torch
        a = np.frombuffer(send, dtype=np.uint8)
        t = self._t(a.astype(np.float64))
        out = [self._t(np.zeros(len(a))) for _ in range(self.ws)]
        self.td.all_gather(out, t)
        return b"".join(np.asarray(o.cpu().numpy(), dtype=np.uint8).tobytes() for o in out)

    def broadcast_bytes(self, b: bytes, n: int) -> bytes:
        if self.ws == 1:
            return b
        t = self._t(np.frombuffer(b, dtype=np.uint8).astype(np.float64) if self.rank == 0 else np.zeros(n))
        self.td.broadcast(t, 0)
        return np.asarray(t.cpu().numpy(), dtype=np.uint8).tobytes()

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
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------ reference (CPU) side
# The unmodified reference compiled from its own headers (oracle/_ref), called
# through thin marshalling wrappers; only the cpu_baseline legs and the
# reference arm use it.
def _ref():
    from oracle_lib import ref
    return ref("mt")


def cpu_cores():
    return os.cpu_count() or 1


def cpu_reference_scene(frames: int, skip: int, root_seed: int = 3):
    """Reference run_scenario (simenv.hpp:239-276), one thread (it is serial):
    plans/s over frames [skip, frames) from its own PlanRecord.wall_seconds."""
    import ctypes as C
    from oracle_lib import PlanRecord, planner_cfg
    r = _ref()
    if r is None:
        return None
    cfg = planner_cfg(max_iters=30, window_carryover=1)
    recs = (PlanRecord * frames)()
    wall = np.zeros(frames)
    assert r.ref_run_scenario(root_seed, 0, frames, C.byref(cfg), recs, wall.ctypes.data_as(C.POINTER(C.c_double))) == 0
    timed = wall[skip:]
    return {"plans_per_s": len(timed) / timed.sum(), "mean_iterations": float(np.mean([recs[i].iterations for i in range(skip, frames)])),
            "frames": len(timed)}


def _parallel_bounded(fn, items, seconds, cores):
    """fn(item) -> work units on `cores` threads until `seconds` pass (ctypes
    releases the GIL); per-thread busy time is summed, so the rate is the
    all-cores rate with every core loaded."""
    done, busy = [0.0] * cores, [0.0] * cores
    t_end = time.perf_counter() + seconds

    def worker(w):
        i = w
        while i < len(items) and time.perf_counter() < t_end:
            t0 = time.perf_counter()
            done[w] += fn(items[i])
            busy[w] += time.perf_counter() - t0
            i += cores
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(worker, range(cores)))
    rate = sum(d / b for d, b in zip(done, busy) if b > 0)
    return rate, sum(done)


def cpu_config5(n_scenes, seconds, cores):
    """Config 5 on the host, scene-parallel: each scene runs the reference's
    run_scenario for 4 frames; frames 1-3 (warm-started, as on the GPU) are
    timed from their own wall_seconds."""
    import ctypes as C
    from oracle_lib import PlanRecord, planner_cfg
    r = _ref()
    cfg = planner_cfg(max_iters=30, window_carryover=1)

    def one(s):
        recs = (PlanRecord * 4)()
        wall = np.zeros(4)
        assert r.ref_run_scenario(s, 0, 4, C.byref(cfg), recs, wall.ctypes.data_as(C.POINTER(C.c_double))) == 0
        one.acc.append(wall[1:].sum())
        return 3
    one.acc = []
    t0 = time.perf_counter()
    _, plans = _parallel_bounded(one, list(range(n_scenes)), seconds, cores)
    wall = time.perf_counter() - t0
    return {"plans_per_s": plans / wall, "plans": int(plans), "cores": cores,
            "sample": f"{int(plans)} warm plans (frames 1-3 of scenes 0..), scene-parallel on {cores} threads, "
                      f"{wall:.1f} s wall"}


def cpu_config1(seconds, cores):
    """Config 1 trials (G=8 N=10 T=1400, BF3, D=30; seeds derive_seed(3003,
    "bench-BF3", t), acceptance.cpp:175), trial-parallel on all cores."""
    import ctypes as C
    import paper_2308_10169_b200 as pe
    from oracle_lib import DEFAULT_GROUP_HYPERS, ptr
    r = _ref()
    hyp = np.ascontiguousarray(DEFAULT_GROUP_HYPERS)

    def one(seed):
        trace, fp, ff = np.zeros(1400), np.zeros(30), C.c_double(0)
        bad = (C.c_size_t * 3)()
        assert r.ref_run_dtpso(3, None, 30, 30.0, 4.0, ptr(hyp), 8, 10, 1400, seed, ptr(trace), ptr(fp), C.byref(ff), bad) == 0
        return 1
    seeds = [pe.derive_seed(3003, "bench-BF3", t) for t in range(4096)]
    t0 = time.perf_counter()
    rate, n = _parallel_bounded(one, seeds, seconds, cores)
    return {"trials_per_s": rate, "trials": int(n), "cores": cores,
            "sample": f"{int(n)} BF3 trials (8x10x1400), trial-parallel on {cores} threads, {time.perf_counter() - t0:.1f} s"}


def cpu_config3(world, seconds, cores):
    """Config 3: lfv_fitness (hsef.hpp:108-119, inner 8x170x30 on the path
    world) candidate-parallel on all cores; an evolution is 80 of them (the
    outer PSO update is negligible)."""
    import ctypes as C
    import paper_2308_10169_b200 as pe
    from oracle_lib import PROB_PATH, ptr, world_from_engine
    r = _ref()
    wb = world_from_engine(world)
    rng = np.random.default_rng(3)
    cands = [np.ascontiguousarray(pe.EVOLVED_PATH_HYPERS.reshape(-1) * rng.uniform(0.8, 1.2, 48)) for _ in range(512)]

    def one(c):
        ws = wb.struct()
        r.ref_lfv_fitness(ptr(c), 8, PROB_PATH, C.byref(ws), 16, 30.0, 4.0, 8, 170, 30, 11)
        return 1
    rate, n = _parallel_bounded(one, cands, seconds, cores)
    return {"ms_per_evolution": 80.0 / rate * 1e3, "lfv_per_s": rate, "cores": cores,
            "sample": f"{int(n)} lfv_fitness runs (8x170x30 path), candidate-parallel on {cores} threads; "
                      f"evolution = 80 runs"}


def cpu_config4(world, seconds, cores, rows=None):
    """Config 4: evaluate_rows (geometry.hpp:262-267) row-parallel on all cores
    over uniform random 64-waypoint rows (a cold swarm's rows are uniform),
    extrapolated to one 65,536-row iteration; the update (6 % of the serial
    time at the paper size) is not included -- declared, a lower bound."""
    import ctypes as C
    from oracle_lib import ptr, world_from_engine, u32p
    r = _ref()
    wb = world_from_engine(world)
    rng = np.random.default_rng(4)
    D = 128
    W = D // 2
    n = rows or cores * 6
    xs = np.concatenate([rng.uniform(0, world.width, (n, W)), rng.uniform(0, world.height, (n, W))], 1)
    chunks = [np.ascontiguousarray(xs[i:i + 1]) for i in range(n)]

    def one(x):
        ws = wb.struct()
        f, q, ln = np.zeros(1), np.zeros(1, dtype=np.uint32), np.zeros(1)
        r.ref_eval_path_rows(C.byref(ws), ptr(x), 1, D, 30.0, 4.0, ptr(f), ptr(q, u32p), ptr(ln))
        return 1
    rate, done = _parallel_bounded(one, chunks, seconds, cores)
    return {"s_per_iteration": 65536.0 / rate, "evals_per_s": rate, "cores": cores,
            "sample": f"{int(done)} random 64-waypoint rows on the config-4 world, row-parallel on {cores} threads, "
                      f"extrapolated to 65,536 rows; fitness only (lower bound on the iteration)"}


# ------------------------------------------------------------------ GPU side
def fused_roofline(kernel, flop_per_launch, ms_per_launch, peak, grid, extra=None):
    achieved = flop_per_launch / (ms_per_launch / 1e3) / 1e12
    d = {"kernel": kernel, "bound": "fp32", "achieved": achieved, "peak": peak,
         "peak_source": "measured FFMA probe (sf_measure_fp32_peak) on this GPU; MEASURED_PEAKS.json has no FP32 entry",
         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
         "traffic": committed_dram_bytes(kernel, grid) if grid else None,
         "traffic_source": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, {PROFILE_CSV}",
         "flop_per_launch": flop_per_launch, "avg_launch_us": 1e3 * ms_per_launch}
    if extra:
        d.update(extra)
    return d


def main():
    a = parse()
    ws, rank, local = dist_env()
    if a.impl == "reference":
        return reference_arm(a, ws, rank)
    import torch
    import paper_2308_10169_b200 as pe
    torch.cuda.set_device(local)
    dist = Dist(ws, rank, local, "nccl")
    eng = pe.Engine(local, a.precision)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    root = 3 + rank
    planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    K, W = a.steps, a.warmup
    scen = [pe.ScenarioConfig(root_seed=root)]
    cores = cpu_cores()
    peak = eng.measure_fp32_peak()
    S, E = planner.dim // 2 + 1, 32
    R2 = planner.groups * planner.per_group

    # ---------------------------------------------------- device-resident value
    sb = pe.SceneBatch(eng, scen, planner, pe.EVOLVED_PATH_HYPERS, W + K)
    sb.run(W)
    eng.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = Clocks(local)
    dist.barrier()
    torch.cuda.synchronize()
    eng.synchronize()
    with torch.cuda.stream(stream):
        for i in range(K):
            flush.zero_()                      # L2 (126 MB) flushed between steps
            evs[i][0].record(stream)
            sb.run(1)
            evs[i][1].record(stream)
    eng.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    dev_ms = dist.max(float(np.sum([e0.elapsed_time(e1) for e0, e1 in evs])))
    recs, _ = sb.records(W, K)
    sb.close()
    iters = np.array([r.iterations for r in recs], dtype=np.float64)
    value = K * ws / (dev_ms / 1e3)
    evals = float(iters.sum()) * R2

    # kernel-only time of the fused planning kernel (same frames, event pair
    # around every launch on the engine stream)
    sb2 = pe.SceneBatch(eng, scen, planner, pe.EVOLVED_PATH_HYPERS, W + K)
    sb2.run(W)
    eng.enable_timing(True)
    for _ in range(K):
        with torch.cuda.stream(stream):
            flush.zero_()
        sb2.run(1)
    k_ms, k_n = eng.kernel_time()
    eng.enable_timing(False)
    recs2, _ = sb2.records(W, K)
    sb2.close()
    flop_launch = float(sum(r.iterations for r in recs2)) * R2 * FLOP_PER_EVAL(S, E) / K
    roof = fused_roofline(LATENCY_KERNEL, flop_launch, k_ms / k_n, peak, "(16, 1, 1)",
                          {"flop_per_eval": FLOP_PER_EVAL(S, E), "launches": int(k_n),
                           "note": "one scene = one 16-CTA cluster on 16 of 148 SMs: latency-bound by construction "
                                   "(DESIGN.md section 4); the throughput measure is the config5 extra"})

    # ------------------------------------------------------------ e2e (host API)
    # sf_run_scenario = run_scenario (simenv.hpp:239-276): per frame
    # sf_plan_frame with HOST world / prev / window and host step_world; L2
    # flushed before every frame outside its wall time
    def e2e_run(engine):
        engine.set_l2_flush(256 * 1024 * 1024)
        dist.barrier()
        rr = engine.run_scenario(scen[0], "sepso", W + K, planner)
        engine.set_l2_flush(0)
        return rr
    recs_e2e = e2e_run(eng)
    h2d, d2h = eng.last_io_bytes()
    e2e_s = dist.max(float(sum(r.wall_seconds for r in recs_e2e[W:])))
    e2e = {"value": K * ws / e2e_s, "unit": "plans/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "timing": "sum of PlanRecord.wall_seconds (host steady_clock around each sf_plan_frame call: validate + "
                     "stage the inputs into pinned host memory + the resident cluster reads them over the bus, plans, "
                     "stores the results into pinned host memory and publishes them + the host reads them; the "
                     "next frame's init walk is launched inside the call, DESIGN.md section 1), frames W..W+K-1",
           "mean_iterations_per_frame": float(np.mean([r.iterations for r in recs_e2e[W:]]))}

    extras = {}
    if not a.no_extra:
        # ---------------------------------------- FP64 parity engine, same frames
        if a.precision == "fp32":
            eng64 = pe.Engine(local, "fp64")
            r64 = e2e_run(eng64)
            eng64.close()
            extras["fp64"] = {"workload": "config2 headline frames through sf_run_scenario, FP64 parity engine "
                                          "(bit-identical to the reference on these frames)",
                              "e2e_plans_per_s": K * ws / dist.max(float(sum(r.wall_seconds for r in r64[W:]))),
                              "mean_iterations_per_frame": float(np.mean([r.iterations for r in r64[W:]]))}
        # ---------------------------------------- Philox stream
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
        extras["philox"] = {"workload": "config2 headline frames, Philox4x32-10 counter stream (different draws, "
                                        "different truncation points)",
                            "plans_per_s": K * ws / (msp / 1e3),
                            "mean_iterations_per_frame": float(np.mean([r.iterations for r in rp]))}
        extras["config5"] = bench_config5(a, eng, dist, stream, flush, planner, peak, cores, torch, pe)
        extras["config4"] = bench_config4(a, eng, dist, peak, cores, pe)
        extras["config3"] = bench_config3(a, eng, dist, peak, cores, pe)
        extras["config1"] = bench_config1(a, eng, dist, cores, pe)
        if dist.rank == 0:
            extras["scale"] = bench_scale(a, eng, pe)

    # ------------------------------------------------------------ CPU baseline
    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        c = cpu_reference_scene(W + K, W)
        if c:
            cpu = {"value": c["plans_per_s"], "unit": "plans/s", "cores": 1, "kind": "reference",
                   "sample": f"reference run_scenario (unmodified, mt19937), root seed 3, frames {W}..{W + K - 1} timed "
                             f"(the reference is serial: 1 thread); mean {c['mean_iterations']:.1f} iterations/frame"}

    if rank == 0:
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
            "vs_baseline": None,
            "vs_baseline_note": "BASELINE.md's C++ figure (15.3 ms/frame) is the 100-frame scenario at 16.2 iterations/"
                                "frame on another box, not these frames; the reference arm times these frames here",
            "dtype": a.precision,
            "data": "synthetic (seeded generate_world scenes; the reference's mt19937_64 draw stream, generated on the device)",
            "config": {"workload": WORKLOAD_C2, "scenes_per_gpu": 1,
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                       "l2": "flushed between steps (256 MiB write)",
                       "mean_iterations_per_frame": float(iters.mean()), "fitness_evals": evals,
                       "evals_per_sec": evals * ws / (dev_ms / 1e3)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # one fused launch per frame (world step included) + the next
            # frame's init walk (prewalk.cu, side stream) launched with it
            "gpu_launches": K + (K - 1 if os.environ.get("SEPSO_PREWALK", "1") != "0" else 0),
            "clocks": clk,
            "host_threads": cores,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    eng.close()
    dist.close()


def bench_config5(a, eng, dist, stream, flush, planner, peak, cores, torch, pe):
    """1,024 independent paper scenes per GPU (scenes sharded by rank, no
    collective), frames 1-3 warm-started, one fused launch per frame."""
    nb = 1024
    rank, ws = dist.rank, dist.ws
    bb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=rank * nb + s) for s in range(nb)], planner,
                       pe.EVOLVED_PATH_HYPERS, 4)
    bb.run(1)
    eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        flush.zero_()
        e0.record(stream)
        bb.run(3)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = dist.max(e0.elapsed_time(e1))
    rb, _ = bb.records(1, 3)
    bb.close()
    iters = float(dist.sum(float(sum(r.iterations for r in rb))))
    S, E = planner.dim // 2 + 1, 32
    R = planner.groups * planner.per_group
    d = {"workload": f"config5: {nb} independent paper scenes per GPU ({nb * ws} total, sharded by rank, no collective), "
                     f"frames 1-3 warm-started, 3 fused launches",
         "plans_per_s": 3 * nb * ws / (ms / 1e3), "n_gpus": ws, "scaling": "weak",
         "mean_iterations": iters / (3 * nb * ws),
         "roofline": {"kernel": "swarm_kernel<float, 1, 1> (throughput launch, 2 CTAs per scene)", "bound": "fp32",
                      "achieved": iters / ws * R * FLOP_PER_EVAL(S, E) / (ms / 1e3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                      "frac": (iters / ws * R * FLOP_PER_EVAL(S, E) / (ms / 1e3) / 1e12) / peak if peak else None,
                      "flop_per_eval": FLOP_PER_EVAL(S, E),
                      "pipes": "ncu FMA / ALU pipe utilisation and issue slots: profiles/r02_swarm_kernel_batched.md"}}
    if dist.rank == 0 and not a.no_cpu_baseline and _ref() is not None:
        c = cpu_config5(4096, a.cpu_seconds, cores)
        d["cpu_baseline"] = {"value": c["plans_per_s"], "unit": "plans/s", "cores": cores, "kind": "reference",
                             "sample": c["sample"]}
    return d


def bench_config4(a, eng, dist, peak, cores, pe):
    """One 65,536-particle swarm (G=8 x N=8192, D=128, 1,024 obstacles) on the
    HBM-staged path; at N>1 its groups are sharded over ranks with one NCCL
    all-gather of the tbest candidates per iteration (sf_plan_frame_sharded)."""
    rank, ws = dist.rank, dist.ws
    sc4 = pe.ScenarioConfig(map_size=366.0 * np.sqrt(128.0), dynamic_obstacles=768, static_obstacles=256, root_seed=1)
    w4 = pe.generate_world(sc4, 1)
    if ws > 1:
        uid = dist.broadcast_bytes(pe.Engine.comm_unique_id() if rank == 0 else bytes(128), 128)
        eng.init_comm(uid, ws, rank)

    def frame4(cap, seed):
        cfg4 = pe.PlannerConfig(groups=8, per_group=8192, dim=128, max_iters_per_frame=cap, auto_truncate=False)
        dist.barrier()
        eng.enable_timing(True)
        rec = eng.plan_frame_sharded(w4, None, pe.EVOLVED_PATH_HYPERS, cfg4, seed)
        ms_, _ = eng.kernel_time()
        eng.enable_timing(False)
        return dist.max(ms_), rec.iterations
    frame4(1, 999)                                                      # warm-up (allocations)
    ms_a, it_a = frame4(2, 1000)
    ms_b, it_b = frame4(6, 1000)
    ms_it = (ms_b - ms_a) / max(1, it_b - it_a)       # steady iteration: K2 + K1 + bests + draws (+ exchange)
    S4, E4 = 65, 4 * w4.n_obstacles
    fl4 = 65536.0 * FLOP_PER_EVAL(S4, E4)
    hbm = measured_peaks().get("hbm_gbs")
    k1_ms, k1_bytes = eng.measure_step_kernel(8, 8192, 128, 5)
    d = {"workload": f"config4: one swarm of 65,536 particles (G=8 x N=8192), D=128, 1,024 obstacles, cold start, "
                     f"iterations 3..6 vs 1..2 (HBM-staged path){'; groups sharded over %d ranks, NCCL all-gather of '
                     'the tbest candidates' % ws if ws > 1 else ''}",
         "ms_per_iteration": ms_it, "init_ms": ms_a - it_a * ms_it, "evals_per_s": 65536.0 / (ms_it / 1e3),
         "n_gpus": ws, "scaling": "strong",
         "roofline_k1": {"kernel": "k_step<float, 4> (TOF update, swarm.hpp:138-174)", "bound": "hbm",
                         "achieved": k1_bytes / (k1_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": (k1_bytes / (k1_ms / 1e3) / 1e9) / hbm if hbm else None,
                         "traffic": committed_dram_bytes("k_step<float, 4>", "(2048, 1, 1)"),
                         "bytes_per_launch": k1_bytes, "avg_launch_us": 1e3 * k1_ms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                         "timing": "CUDA events on the engine stream around [256 MiB L2 eviction + K1] minus around "
                                   "[eviction] alone, mean of 5 (sf_measure_step_kernel)"},
         "roofline_k2": {"kernel": "k_eval_path_wide<float> (+ K1, bests, draws: whole iteration)", "bound": "fp32",
                         "algorithmic_tflops": fl4 / (ms_it / 1e3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                         "note": "the algorithmic count (every segment x edge pair, SURVEY.md 8(d)) over a kernel whose "
                                 "map grid and box cull skip most pairs: a rate, not a pipe fraction; the pipe "
                                 "utilisation of the executed pair tests is in profiles/r02_k_eval_path_wide_config4.md"}}
    if rank == 0 and not a.no_cpu_baseline and _ref() is not None:
        c = cpu_config4(w4, a.cpu_seconds, cores)
        d["cpu_baseline"] = {"value": c["s_per_iteration"], "unit": "s/iteration", "cores": cores, "kind": "reference",
                             "sample": c["sample"]}
    return d


def bench_config3(a, eng, dist, peak, cores, pe):
    """HSEF (hsef.hpp:125-171): outer PSO (8 x 10) over inner 8 x 170 x 30 path
    swarms on the frozen frame-0 world; the 80 candidates of an evolution run in
    one launch, split over ranks (host all-gather of the LFVs, outer PSO
    replicated with the same seed)."""
    rank, ws = dist.rank, dist.ws
    w3 = pe.generate_world(pe.ScenarioConfig(root_seed=3), pe.derive_seed(3, "world"))
    if ws > 1:
        eng.set_exchange(ws, rank, dist.allgather_bytes)
    eng.evolve("path", (8, 170, 30), (8, 10, 1), 40, world=w3, dim=16)          # warm-up
    dist.barrier()
    t0 = time.perf_counter()
    eng.evolve("path", (8, 170, 30), (8, 10, 3), 41, world=w3, dim=16)
    dt = dist.max(time.perf_counter() - t0)
    if ws > 1:
        eng.set_exchange(1, 0, None)
    ms_ev = dt / 3 * 1e3
    flop = 80 * 8 * 170 * 30 * FLOP_PER_EVAL(9, 32)
    d = {"workload": "config3: HSEF evolve, inner (8,170,30) path on the frame-0 paper world, outer (8,10), 3 "
                     f"evolutions timed (wall, host API){'; candidates split over %d ranks' % ws if ws > 1 else ''}",
         "ms_per_evolution": ms_ev, "inner_evals_per_s": 80 * 1360 * 30 / (ms_ev / 1e3), "n_gpus": ws,
         "scaling": "strong",
         "roofline": {"kernel": "swarm_kernel<float, 1, 1> (80 inner swarms, one launch per evolution)", "bound": "fp32",
                      "achieved": flop / (ms_ev / 1e3) / 1e12 / ws, "peak": peak, "unit": "TFLOP/s",
                      "frac": flop / (ms_ev / 1e3) / 1e12 / ws / peak if peak else None,
                      "note": "per GPU, whole evolution wall time (host outer PSO included)"}}
    if rank == 0 and not a.no_cpu_baseline and _ref() is not None:
        c = cpu_config3(w3, a.cpu_seconds, cores)
        d["cpu_baseline"] = {"value": c["ms_per_evolution"], "unit": "ms/evolution", "cores": cores,
                             "kind": "reference", "sample": c["sample"]}
    return d


def bench_config1(a, eng, dist, cores, pe):
    """1,024 BF3 trials per GPU (G=8 x N=10 x T=1400, D=30), trials sharded by
    rank, one batched launch through the public API (host buffers)."""
    rank, ws = dist.rank, dist.ws
    seeds = np.array([pe.derive_seed(3003, "bench-BF3", rank * 1024 + t) for t in range(1024)], dtype=np.uint64)
    eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)     # warm-up, same size
    dist.barrier()
    t0 = time.perf_counter()
    eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)
    dt = dist.max(time.perf_counter() - t0)
    d = {"workload": f"config1: 1,024 BF3 trials per GPU ({1024 * ws} total, sharded by rank), G=8 N=10 T=1400 D=30, "
                     "one batched call (wall, host API)",
         "trials_per_s": 1024 * ws / dt, "evals_per_s": 1024 * ws * 80 * 1400 / dt, "n_gpus": ws, "scaling": "weak"}
    if rank == 0 and not a.no_cpu_baseline and _ref() is not None:
        c = cpu_config1(a.cpu_seconds, cores)
        d["cpu_baseline"] = {"value": c["trials_per_s"], "unit": "trials/s", "cores": cores, "kind": "reference",
                             "sample": c["sample"]}
    return d


def bench_scale(a, eng, pe):
    """The reference's `scale` harness shape (proj/tools/swarmforge.cpp:186-255:
    BF1, G=8, N=16,384, D=1,000, T=10 -- 131,072 particles of 1,000 dims, the
    HBM-staged path): the engine's run_dtpso wall time through the host API,
    beside the reference's batched run_dtpso and its per-particle oracle
    run_dppso_reference (runner.hpp:135-239), each timed for T=1 on this host
    and extrapolated to T=10 (declared)."""
    import ctypes as C
    G, N, D, T = 8, 16384, 1000, 10
    eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, 2, 1, dim=D)         # warm-up (arena)
    t0 = time.perf_counter()
    eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, T, 1, dim=D)
    gpu_s = time.perf_counter() - t0
    d = {"workload": "scale harness: BF1, G=8 N=16384 D=1000 T=10 (131,072 particles), run_dtpso through the host API",
         "gpu_seconds": gpu_s, "evals_per_s": G * N * T / gpu_s}
    r = _ref()
    if r is not None and not a.no_cpu_baseline:
        from oracle_lib import ptr            # CPU baseline only: the reference's ctypes helpers
        h = np.ascontiguousarray(pe.DEFAULT_GROUP_HYPERS)
        bad = (C.c_size_t * 3)()

        def batched(t):
            tr, fp, ff = np.zeros(t), np.zeros(D), C.c_double(0)
            t0 = time.perf_counter()
            r.ref_run_dtpso(1, None, D, 30.0, 4.0, ptr(h), G, N, t, 1, ptr(tr), ptr(fp), C.byref(ff), bad)
            return time.perf_counter() - t0

        def per_particle(t):
            tr, fp, ff, wall = np.zeros(t), np.zeros(D), C.c_double(0), C.c_double(0)
            r.ref_run_dppso_reference(1, None, D, 30.0, 4.0, ptr(h), G, N, t, 1, ptr(tr), ptr(fp), C.byref(ff),
                                      C.byref(wall))
            return wall.value
        b1, b2 = batched(1), batched(2)
        p1, p2 = per_particle(1), per_particle(2)
        how = "one thread, T=1 and T=2 timed, extrapolated to T=10 as t1 + 9 (t2 - t1) (declared)"
        d["cpu_baseline"] = {"value": b1 + 9 * (b2 - b1), "unit": "s", "cores": 1, "kind": "reference",
                             "sample": f"reference run_dtpso (batched), {how}"}
        d["cpu_per_particle_oracle"] = {"value": p1 + 9 * (p2 - p1), "unit": "s", "cores": 1, "kind": "reference",
                                        "sample": f"reference run_dppso_reference (per-particle oracle), {how}; "
                                                  "published on the author's box: 11.06 s batched vs 8.71 s "
                                                  "per-particle (proj/test_output.txt:10)"}
    return d


def reference_arm(a, ws, rank):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    headers) on the headline workload and frames, on this box's host."""
    if rank != 0:
        return 0
    if _ref() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsfref_mt.so not built"}))
        return 0
    K, W = a.steps, a.warmup
    c = cpu_reference_scene(W + K, W)
    value = c["plans_per_s"]
    line = {"impl": "reference", "metric": "plans_per_sec", "value": value, "unit": "plans/s",
            "n_gpus": a.gpus, "steps": K, "warmup": W, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64",
            "data": "synthetic", "config": {"workload": WORKLOAD_C2, "mean_iterations_per_frame": c["mean_iterations"]},
            "cpu_baseline": {"value": value, "unit": "plans/s", "cores": 1, "kind": "reference",
                             "sample": f"reference run_scenario root seed 3, frames {W}..{W + K - 1} timed from its own "
                                       f"PlanRecord.wall_seconds; the reference is serial (1 thread)"},
            "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
