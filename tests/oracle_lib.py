"""ctypes bindings to the CPU checkers -- TEST INFRASTRUCTURE ONLY.

* ``oracle()``  -> oracle/liboracle.so, the C restatement of the reference hot path.
* ``ref(kind)`` -> oracle/_ref/libsfref_{mt,philox}.so, the reference compiled
  unmodified from its own headers (``mt`` = as shipped, ``philox`` = with the
  shared-RNG shim).  ``None`` when it was not built (no /root/reference).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may use
this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")

RNG_MT, RNG_PHILOX = 0, 1
PROB_PATH, PROB_SPHERE, PROB_ROSENBROCK, PROB_RASTRIGIN, PROB_GRIEWANK, PROB_ACKLEY = range(6)

dp = C.POINTER(C.c_double)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
szp = C.POINTER(C.c_size_t)


class World(C.Structure):
    _fields_ = [("width", C.c_double), ("height", C.c_double),
                ("start", C.c_double * 2), ("target", C.c_double * 2),
                ("start_vel", C.c_double * 2), ("target_vel", C.c_double * 2),
                ("n_obstacles", C.c_size_t), ("offsets", u32p), ("verts", dp),
                ("obs_vel", dp)]


class PlannerCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("delta", C.c_double), ("tw", C.c_size_t), ("pi_radius", C.c_double),
                ("max_iters", C.c_size_t), ("G", C.c_size_t), ("N", C.c_size_t),
                ("D", C.c_size_t), ("auto_truncate", C.c_int),
                ("window_carryover", C.c_int)]


class PlanRecord(C.Structure):
    _fields_ = [("fitness", C.c_double), ("length", C.c_double),
                ("intersections", C.c_size_t), ("iterations", C.c_size_t),
                ("truncated", C.c_int), ("collision_free", C.c_int)]


class ScenarioCfg(C.Structure):
    _fields_ = [("map_size", C.c_double), ("dynamic_obstacles", C.c_size_t),
                ("static_obstacles", C.c_size_t), ("min_side", C.c_double),
                ("max_side", C.c_double), ("max_speed", C.c_double),
                ("start_speed", C.c_double), ("target_speed", C.c_double),
                ("dt", C.c_double)]


def ptr(a, t=dp):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def planner_cfg(**kw) -> PlannerCfg:
    """PlannerConfig defaults (planner.hpp:19-35)."""
    d = dict(alpha=30.0, beta=4.0, gamma=0.25, delta=10.0, tw=20, pi_radius=20.0,
             max_iters=50, G=8, N=170, D=16, auto_truncate=1, window_carryover=0)
    d.update(kw)
    return PlannerCfg(**d)


def scenario_cfg(**kw) -> ScenarioCfg:
    """ScenarioConfig defaults (simenv.hpp:17-28)."""
    d = dict(map_size=366.0, dynamic_obstacles=6, static_obstacles=2, min_side=30.0,
             max_side=80.0, max_speed=5.0, start_speed=3.0, target_speed=8.0, dt=1.0)
    d.update(kw)
    return ScenarioCfg(**d)


class WorldBuf:
    """Owns the numpy buffers behind a ``World`` struct."""

    def __init__(self, width, height, start, target, polys, start_vel=(0, 0),
                 target_vel=(0, 0), vels=None):
        self.head = np.array([width, height, *start, *target, *start_vel, *target_vel],
                             dtype=np.float64)
        self.offsets = np.zeros(len(polys) + 1, dtype=np.uint32)
        for i, p in enumerate(polys):
            self.offsets[i + 1] = self.offsets[i] + len(p)
        self.verts = (np.concatenate([np.asarray(p, dtype=np.float64).reshape(-1)
                                      for p in polys]) if polys
                      else np.zeros(2, dtype=np.float64))
        self.vel = (np.asarray(vels, dtype=np.float64).reshape(-1).copy() if vels is not None
                    else np.zeros(2 * max(len(polys), 1), dtype=np.float64))
        self.n = len(polys)

    def struct(self) -> World:
        h = self.head
        return World(h[0], h[1], (C.c_double * 2)(h[2], h[3]), (C.c_double * 2)(h[4], h[5]),
                     (C.c_double * 2)(h[6], h[7]), (C.c_double * 2)(h[8], h[9]),
                     self.n, ptr(self.offsets, u32p), ptr(self.verts), ptr(self.vel))

    def polys(self):
        return [self.verts[2 * self.offsets[i]:2 * self.offsets[i + 1]].reshape(-1, 2)
                for i in range(self.n)]

    def copy(self):
        w = WorldBuf.__new__(WorldBuf)
        w.head, w.offsets, w.verts, w.vel, w.n = (self.head.copy(), self.offsets.copy(),
                                                  self.verts.copy(), self.vel.copy(), self.n)
        return w


def rect(x0, y0, x1, y1):
    return [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_cache: dict = {}


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, "oracle"], check=True)


def oracle():
    if "oracle" in _cache:
        return _cache["oracle"]
    path = os.path.join(ORACLE_DIR, "liboracle.so")
    if not os.path.exists(path):
        build_oracle()
    lib = C.CDLL(path)
    W = C.POINTER(World)
    _sig(lib, "or_derive_seed", C.c_uint64, [C.c_uint64, C.c_char_p])
    _sig(lib, "or_derive_seed_idx", C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint64])
    _sig(lib, "or_philox4x32_10", None, [u32p, u32p, u32p])
    _sig(lib, "or_philox_word", C.c_uint64, [C.c_uint64, C.c_uint64])
    _sig(lib, "or_mt_nth", C.c_uint64, [C.c_uint64, C.c_uint64])
    _sig(lib, "or_segments_intersect", C.c_int, [dp, dp, dp, dp])
    _sig(lib, "or_point_strictly_inside", C.c_int, [dp, dp, C.c_size_t])
    _sig(lib, "or_count_intersections", C.c_size_t, [dp, C.c_size_t, W])
    _sig(lib, "or_path_length", C.c_double, [dp, C.c_size_t, W])
    _sig(lib, "or_eval_path_rows", None,
         [dp, C.c_size_t, C.c_size_t, W, C.c_double, C.c_double, dp, u32p])
    _sig(lib, "or_bench_eval", C.c_double, [C.c_int, dp, C.c_size_t])
    _sig(lib, "or_should_truncate", C.c_int, [dp, C.c_size_t, C.c_int, C.POINTER(PlannerCfg)])
    _sig(lib, "or_plan_frame", C.c_int,
         [W, dp, dp, C.POINTER(PlannerCfg), C.c_uint64, C.c_int, dp, szp,
          C.POINTER(PlanRecord), dp, szp])
    _sig(lib, "or_unflatten", None, [dp, C.c_size_t, dp])
    _sig(lib, "or_generate_world", C.c_int,
         [C.POINTER(ScenarioCfg), C.c_uint64, C.c_int, dp, u32p, dp, dp, u8p])
    _sig(lib, "or_step_world", None, [dp, C.c_size_t, u32p, dp, dp, C.c_double])
    _sig(lib, "or_init_swarm_seed", C.c_int,
         [dp, dp, dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int, dp, C.c_size_t,
          C.c_double, dp, dp])
    _sig(lib, "or_step_seed", C.c_int,
         [dp, dp, dp, C.c_size_t, C.c_size_t, C.c_size_t, dp, dp, dp, dp, dp, C.c_uint64, C.c_int,
          C.c_uint64, C.c_size_t, C.c_size_t])
    _sig(lib, "or_update_bests_arrays", None,
         [C.c_size_t, C.c_size_t, C.c_size_t, dp, dp, dp, dp, dp, dp, dp, dp])
    _sig(lib, "or_run_dtpso_flat", C.c_int,
         [C.c_int, W, C.c_size_t, dp, dp, C.c_double, C.c_double, dp, C.c_size_t, C.c_size_t,
          C.c_size_t, C.c_uint64, C.c_int, dp, dp, dp, szp])
    _sig(lib, "or_lfv_flat", C.c_double,
         [dp, C.c_size_t, C.c_int, W, C.c_size_t, dp, dp, C.c_double, C.c_double, C.c_size_t,
          C.c_size_t, C.c_size_t, C.c_uint64, C.c_int])
    _sig(lib, "or_evolve_flat", C.c_int,
         [C.c_int, W, C.c_size_t, dp, dp, C.c_double, C.c_double, C.c_size_t, C.c_size_t,
          C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, dp, C.c_int, dp, dp, dp])
    _cache["oracle"] = lib
    return lib


def ref(kind: str = "philox"):
    key = "ref_" + kind
    if key in _cache:
        return _cache[key]
    path = os.path.join(ORACLE_DIR, "_ref", f"libsfref_{kind}.so")
    if not os.path.exists(path):
        _cache[key] = None
        return None
    lib = C.CDLL(path)
    W = C.POINTER(World)
    _sig(lib, "ref_uniform_stream", None, [C.c_uint64, C.c_uint64, dp])
    _sig(lib, "ref_derive_seed", C.c_uint64, [C.c_uint64, C.c_char_p])
    _sig(lib, "ref_derive_seed_idx", C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint64])
    _sig(lib, "ref_init_swarm", C.c_int,
         [dp, C.c_size_t, C.c_size_t, C.c_size_t, dp, dp, C.c_uint64, dp, dp])
    _sig(lib, "ref_step", C.c_int,
         [C.c_size_t, C.c_size_t, C.c_size_t, dp, dp, dp, dp, dp, dp, dp, dp, C.c_uint64,
          C.c_uint64, C.c_size_t, C.c_size_t])
    _sig(lib, "ref_update_bests", None,
         [C.c_size_t, C.c_size_t, C.c_size_t, dp, dp, dp, dp, dp, dp, dp, dp])
    _sig(lib, "ref_segments_intersect", C.c_int, [dp, dp, dp, dp])
    _sig(lib, "ref_point_strictly_inside", C.c_int, [dp, dp, C.c_size_t])
    _sig(lib, "ref_eval_path_rows", None,
         [W, dp, C.c_size_t, C.c_size_t, C.c_double, C.c_double, dp, u32p, dp])
    _sig(lib, "ref_bench_eval", C.c_int, [C.c_int, dp, C.c_size_t, C.c_size_t, dp])
    _sig(lib, "ref_run_dtpso", C.c_int,
         [C.c_int, W, C.c_size_t, C.c_double, C.c_double, dp, C.c_size_t, C.c_size_t,
          C.c_size_t, C.c_uint64, dp, dp, dp, szp])
    _sig(lib, "ref_run_dppso_reference", C.c_int,
         [C.c_int, W, C.c_size_t, C.c_double, C.c_double, dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64,
          dp, dp, dp, dp])
    _sig(lib, "ref_run_pso_reference", C.c_int,
         [C.c_int, W, C.c_size_t, C.c_double, C.c_double, C.c_size_t, C.c_size_t, C.c_uint64, dp, dp, dp, dp])
    _sig(lib, "ref_priori_init", C.c_int,
         [dp, dp, C.POINTER(PlannerCfg), dp, dp, C.c_uint64, dp, dp])
    _sig(lib, "ref_should_truncate", C.c_int, [dp, C.c_size_t, C.c_int, C.POINTER(PlannerCfg)])
    _sig(lib, "ref_plan_frame", C.c_int,
         [W, dp, dp, C.POINTER(PlannerCfg), C.c_uint64, dp, szp, C.POINTER(PlanRecord), dp,
          szp])
    _sig(lib, "ref_run_scenario", C.c_int,
         [C.c_uint64, C.c_int, C.c_size_t, C.POINTER(PlannerCfg), C.POINTER(PlanRecord), dp])
    _sig(lib, "ref_unflatten", None, [dp, C.c_size_t, dp])
    _sig(lib, "ref_lfv_fitness", C.c_double,
         [dp, C.c_size_t, C.c_int, W, C.c_size_t, C.c_double, C.c_double, C.c_size_t,
          C.c_size_t, C.c_size_t, C.c_uint64])
    _sig(lib, "ref_evolve", C.c_int,
         [C.c_int, W, C.c_size_t, C.c_double, C.c_double, C.c_size_t, C.c_size_t,
          C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, dp, dp, dp, dp])
    _sig(lib, "ref_generate_world", C.c_int,
         [C.POINTER(ScenarioCfg), C.c_uint64, dp, u32p, dp, dp, u8p])
    _sig(lib, "ref_step_world", None, [dp, C.c_size_t, u32p, dp, dp, C.c_double])
    _cache[key] = lib
    return lib


# ---------------------------------------------------------------- helpers --
DEFAULT_GROUP_HYPERS = np.array([   # hypers.hpp:51-63
    [2, 1, 1, 0.4, 0.2, 0.2], [1, 1, 2, 0.7, 0.3, 0.1], [2, 2, 1, 0.8, 0.1, 0.6],
    [2, 2, 1, 0.8, 0.6, 0.4], [2, 1, 2, 0.2, 0.1, 0.3], [2, 1, 2, 0.9, 0.5, 0.5],
    [1, 2, 2, 0.4, 0.1, 0.8], [1, 2, 2, 0.9, 0.3, 0.3]], dtype=np.float64)
EVOLVED_PATH_HYPERS = np.array([    # hypers.hpp:75-87
    [1.53, 1.29, 1.34, 0.48, 0.19, 0.35], [1.72, 1.53, 1.34, 0.73, 0.28, 0.32],
    [1.34, 1.42, 1.33, 0.48, 0.21, 0.62], [1.76, 1.60, 1.21, 0.47, 0.30, 0.63],
    [1.68, 1.27, 1.25, 0.73, 0.36, 0.41], [1.66, 1.54, 1.54, 0.39, 0.16, 0.45],
    [1.57, 1.48, 1.75, 0.56, 0.34, 0.38], [1.31, 1.71, 1.23, 0.36, 0.25, 0.50]],
    dtype=np.float64)


def generate_world(lib_kind="oracle", seed=1, rng=RNG_PHILOX, **cfg_kw) -> WorldBuf:
    c = scenario_cfg(**cfg_kw)
    n = c.dynamic_obstacles + c.static_obstacles
    head = np.zeros(10)
    offsets = np.zeros(n + 1, dtype=np.uint32)
    verts = np.zeros(8 * n)
    vel = np.zeros(2 * n)
    kinds = np.zeros(n, dtype=np.uint8)
    if lib_kind == "oracle":
        st = oracle().or_generate_world(C.byref(c), seed, rng, ptr(head), ptr(offsets, u32p),
                                        ptr(verts), ptr(vel), ptr(kinds, u8p))
    else:
        st = ref(lib_kind).ref_generate_world(C.byref(c), seed, ptr(head), ptr(offsets, u32p),
                                              ptr(verts), ptr(vel), ptr(kinds, u8p))
    assert st == 0
    w = WorldBuf.__new__(WorldBuf)
    w.head, w.offsets, w.verts, w.vel, w.n = head, offsets, verts, vel, n
    return w


def oracle_plan_frame(world: WorldBuf, prev, hypers, cfg: PlannerCfg, seed, rng=RNG_PHILOX,
                      window=None):
    """Returns (status, record, best_particle, window_out)."""
    o = oracle()
    D = cfg.D
    best = np.zeros(D)
    rec = PlanRecord()
    wl = C.c_size_t(0 if window is None else len(window))
    wbuf = np.zeros(max(int(wl.value), cfg.tw) + 2)
    if window is not None:
        wbuf[:len(window)] = window
    bad = (C.c_size_t * 3)()
    hyp = np.ascontiguousarray(hypers, dtype=np.float64)
    prev_a = None if prev is None else np.ascontiguousarray(prev, dtype=np.float64)
    st = o.or_plan_frame(C.byref(world.struct()), ptr(prev_a), ptr(hyp), C.byref(cfg), seed,
                         rng, ptr(wbuf), C.byref(wl), C.byref(rec), ptr(best), bad)
    return st, rec, best, wbuf[:wl.value].copy(), tuple(bad)


def ref_plan_frame(kind, world: WorldBuf, prev, hypers, cfg: PlannerCfg, seed, window=None):
    r = ref(kind)
    D = cfg.D
    best = np.zeros(D)
    rec = PlanRecord()
    wl = C.c_size_t(0 if window is None else len(window))
    wbuf = np.zeros(max(int(wl.value), cfg.tw) + 2)
    if window is not None:
        wbuf[:len(window)] = window
    bad = (C.c_size_t * 3)()
    hyp = np.ascontiguousarray(hypers, dtype=np.float64)
    prev_a = None if prev is None else np.ascontiguousarray(prev, dtype=np.float64)
    st = r.ref_plan_frame(C.byref(world.struct()), ptr(prev_a), ptr(hyp), C.byref(cfg), seed,
                          ptr(wbuf), C.byref(wl), C.byref(rec), ptr(best), bad)
    return st, rec, best, wbuf[:wl.value].copy(), tuple(bad)


def world_from_engine(pw) -> WorldBuf:
    """oracle WorldBuf from a paper_2308_10169_b200.PolygonWorld (same doubles)."""
    w = WorldBuf(pw.width, pw.height, pw.start, pw.target, pw.obstacles(), pw.start_velocity,
                 pw.target_velocity, pw.velocities[:pw.n_obstacles] if pw.n_obstacles else None)
    return w


def float_world(pw):
    """The FP32 engine plans on the FP32-rounded world; give the oracle the same."""
    import paper_2308_10169_b200 as pe
    r = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    return pe.PolygonWorld(float(np.float32(pw.width)), float(np.float32(pw.height)), r(pw.start),
                           r(pw.target), [r(p) for p in pw.obstacles()], pw.start_velocity,
                           pw.target_velocity, pw.velocities)


def oracle_run_dtpso(kind, hypers, G, N, T, seed, D=30, lo=None, hi=None, world=None,
                     alpha=30.0, beta=4.0, rng=RNG_PHILOX):
    o = oracle()
    trace = np.zeros(T)
    fp = np.zeros(D)
    ff = C.c_double(0)
    bad = (C.c_size_t * 3)()
    lo_a = None if lo is None else np.ascontiguousarray(lo, dtype=np.float64)
    hi_a = None if hi is None else np.ascontiguousarray(hi, dtype=np.float64)
    wb = world_from_engine(world) if world is not None else None
    ws = C.byref(wb.struct()) if wb is not None else None
    hyp = np.ascontiguousarray(hypers, dtype=np.float64)
    st = o.or_run_dtpso_flat(kind, ws, D, ptr(lo_a), ptr(hi_a), alpha, beta, ptr(hyp), G, N, T,
                             seed, rng, ptr(trace), ptr(fp), C.byref(ff), bad)
    return st, trace, fp, ff.value, tuple(bad)
