"""Python mirror of the reference planner API over the C ABI (include/sepso.h).

The product is ``lib/libsepso_cuda.so`` (CUDA kernels for sm_100a + the host
C++ runtime).  This module only marshals arguments: there is no Python or CPU
compute path, and importing it on a machine without the built library raises.

Names follow the reference (proj/include/swarmforge/): ``PlannerConfig``,
``PolygonWorld``, ``PlanRecord``, ``plan_frame``, ``run_dtpso``, ``lfv_fitness``,
``evolve``, ``generate_world``, ``step_world``, ``run_scenario``; errors map to
``ValueError`` (std::invalid_argument) and ``NonFiniteFitnessError``
(runner.hpp:19-33).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEPSO_LIB") or os.path.join(_HERE, "lib", "libsepso_cuda.so")

SF_OK, SF_INVALID_ARGUMENT, SF_NON_FINITE, SF_CUDA_ERROR, SF_UNSUPPORTED, SF_RUNTIME_ERROR = range(6)
FP32, FP64 = 0, 1
PROBLEMS = {"path": 0, "BF1": 1, "BF2": 2, "BF3": 3, "BF4": 4, "ACKLEY": 5,
            "sphere": 1, "rosenbrock": 2, "rastrigin": 3, "griewank": 4, "ackley": 5}
VARIANTS = ["sepso", "sepso-noat", "sepso-nopi", "dtpso", "dppso", "pso"]

# C ABI entry points (the symbols tests/test_abi.py checks against include/sepso.h)
ABI_SYMBOLS = [
    "sf_abi_version", "sf_last_error", "sf_ctx_create", "sf_ctx_destroy", "sf_ctx_precision",
    "sf_ctx_stream", "sf_ctx_synchronize", "sf_ctx_set_launch", "sf_ctx_enable_timing",
    "sf_ctx_kernel_time", "sf_plan_frame", "sf_plan_frames_batched", "sf_run_dtpso",
    "sf_run_dtpso_batched", "sf_lfv_batch", "sf_evolve", "sf_init_swarm", "sf_step",
    "sf_update_bests", "sf_eval_path_rows", "sf_eval_bench_rows", "sf_should_truncate",
    "sf_generate_world", "sf_step_world", "sf_run_scenario", "sf_scene_batch_create",
    "sf_scene_batch_run", "sf_scene_batch_records", "sf_scene_batch_destroy",
    "sf_ctx_last_io_bytes", "sf_measure_fp32_peak", "sf_ctx_set_l2_flush",
    "sf_comm_unique_id", "sf_ctx_init_comm", "sf_plan_frame_sharded", "sf_ctx_set_rng",
    "sf_ctx_rng", "sf_mt_jump_poly", "sf_derive_seed", "sf_measure_step_kernel", "sf_ctx_set_exchange",
    "sf_ctx_hint_next_seed",
]
# sf_allgather_fn: int (*)(void* user, const void* send, void* recv, size_t bytes)
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
RNGS = {"philox": 0, "mt19937": 1}


class NonFiniteFitnessError(RuntimeError):
    """runner.hpp:19-33 -- names the offending particle (group, index, iteration)."""

    def __init__(self, group, index, iteration, msg=""):
        super().__init__(msg or f"non-finite fitness for particle ({group},{index}) at iteration {iteration}")
        self.group, self.index_in_group, self.iteration = int(group), int(index), int(iteration)


class CudaError(RuntimeError):
    pass


# ------------------------------------------------------------------ structs
class _Point(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double)]


class _World(C.Structure):
    _fields_ = [("width", C.c_double), ("height", C.c_double), ("start", _Point),
                ("target", _Point), ("start_velocity", _Point), ("target_velocity", _Point),
                ("n_obstacles", C.c_uint32), ("vertex_offsets", C.POINTER(C.c_uint32)),
                ("vertices", C.POINTER(_Point)), ("velocities", C.POINTER(_Point))]


class _PlannerCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("delta", C.c_double), ("tw", C.c_uint32), ("pi_radius", C.c_double),
                ("max_iters_per_frame", C.c_uint32), ("groups", C.c_uint32),
                ("per_group", C.c_uint32), ("dim", C.c_uint32), ("auto_truncate", C.c_int32),
                ("window_carryover", C.c_int32)]


class _PlanRecord(C.Structure):
    _fields_ = [("fitness", C.c_double), ("length", C.c_double),
                ("intersections", C.c_uint32), ("iterations", C.c_uint32),
                ("truncated", C.c_int32), ("collision_free", C.c_int32),
                ("wall_seconds", C.c_double)]


class _Problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_uint32), ("lo", C.POINTER(C.c_double)),
                ("hi", C.POINTER(C.c_double)), ("world", C.POINTER(_World)),
                ("alpha", C.c_double), ("beta", C.c_double)]


class _ScenarioCfg(C.Structure):
    _fields_ = [("map_size", C.c_double), ("dynamic_obstacles", C.c_uint32),
                ("static_obstacles", C.c_uint32), ("min_side", C.c_double),
                ("max_side", C.c_double), ("max_speed", C.c_double),
                ("start_speed", C.c_double), ("target_speed", C.c_double),
                ("frames", C.c_uint32), ("dt", C.c_double), ("root_seed", C.c_uint64)]


_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


_LIB = None


def lib():
    """Load the engine library; raise loudly when it has not been built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"SEPSO CUDA engine not built: {LIB_PATH} is missing "
                           "(run __graft_entry__.build() or `make -C paper_2308_10169_b200`)")
    L = C.CDLL(LIB_PATH)
    W, P, Pr = C.POINTER(_World), C.POINTER(_PlannerCfg), C.POINTER(_PlanRecord)
    sig = {
        "sf_abi_version": (C.c_int, []),
        "sf_derive_seed": (C.c_uint64, [C.c_uint64, C.c_char_p, C.c_size_t, C.c_int, C.c_uint64]),
        "sf_last_error": (C.c_char_p, []),
        "sf_ctx_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
        "sf_ctx_destroy": (C.c_int, [C.c_void_p]),
        "sf_ctx_precision": (C.c_int, [C.c_void_p]),
        "sf_ctx_stream": (C.c_void_p, [C.c_void_p]),
        "sf_ctx_synchronize": (C.c_int, [C.c_void_p]),
        "sf_ctx_set_launch": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
        "sf_ctx_set_rng": (C.c_int, [C.c_void_p, C.c_int]),
        "sf_ctx_rng": (C.c_int, [C.c_void_p]),
        "sf_ctx_enable_timing": (C.c_int, [C.c_void_p, C.c_int]),
        "sf_ctx_kernel_time": (C.c_int, [C.c_void_p, _dp, _u64p]),
        "sf_plan_frame": (C.c_int, [C.c_void_p, W, _dp, _dp, P, C.c_uint64, _dp, _u32p,
                                    C.c_uint32, Pr, _dp, _u64p]),
        "sf_plan_frames_batched": (C.c_int, [C.c_void_p, C.c_uint32, W, _dp, _u8p, _dp, P, _u64p,
                                             _dp, _u32p, Pr, _dp, _i32p, _u64p]),
        "sf_run_dtpso": (C.c_int, [C.c_void_p, C.POINTER(_Problem), _dp, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_uint64, _dp, _dp, _dp, _u64p]),
        "sf_run_dtpso_batched": (C.c_int, [C.c_void_p, C.POINTER(_Problem), C.c_uint32, _dp,
                                           C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, _u64p,
                                           _dp, _dp, _dp, _i32p]),
        "sf_lfv_batch": (C.c_int, [C.c_void_p, C.POINTER(_Problem), C.c_uint32, _dp, _u64p,
                                   C.c_uint32, C.c_uint32, C.c_uint32, _dp]),
        "sf_evolve": (C.c_int, [C.c_void_p, C.POINTER(_Problem), C.c_uint32, C.c_uint32,
                                C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _dp,
                                _dp, _dp, _dp, C.c_void_p, C.c_void_p]),
        "sf_init_swarm": (C.c_int, [C.c_void_p, _dp, _dp, _dp, C.c_uint32, C.c_uint32,
                                    C.c_uint32, C.c_uint64, C.c_uint64, _dp, C.c_uint32, C.c_double,
                                    _dp, _dp]),
        "sf_step": (C.c_int, [C.c_void_p, _dp, _dp, _dp, C.c_uint32, C.c_uint32, C.c_uint32, _dp,
                              _dp, _dp, _dp, _dp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]),
        "sf_update_bests": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, _dp, _dp,
                                      _dp, _dp, _dp, _dp, _dp, _dp]),
        "sf_eval_path_rows": (C.c_int, [C.c_void_p, W, _dp, C.c_uint32, C.c_uint32, C.c_double,
                                        C.c_double, _dp, _u32p]),
        "sf_eval_bench_rows": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_uint32, C.c_uint32, _dp]),
        "sf_should_truncate": (C.c_int, [_dp, C.c_uint32, C.c_int, P, C.POINTER(C.c_int)]),
        "sf_generate_world": (C.c_int, [C.POINTER(_ScenarioCfg), C.c_uint64, C.c_int, W, _u32p,
                                        C.POINTER(_Point), C.POINTER(_Point)]),
        "sf_step_world": (C.c_int, [W, C.POINTER(_Point), C.POINTER(_Point), C.c_double]),
        "sf_run_scenario": (C.c_int, [C.c_void_p, C.POINTER(_ScenarioCfg), C.c_int, C.c_uint32,
                                      P, _dp, C.c_uint32, Pr, _dp]),
        "sf_scene_batch_create": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(_ScenarioCfg), P,
                                            _dp, C.c_uint32, C.POINTER(C.c_void_p)]),
        "sf_scene_batch_run": (C.c_int, [C.c_void_p, C.c_uint32]),
        "sf_scene_batch_records": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, Pr, _dp]),
        "sf_scene_batch_destroy": (C.c_int, [C.c_void_p]),
        "sf_ctx_last_io_bytes": (C.c_int, [C.c_void_p, _u64p, _u64p]),
        "sf_measure_fp32_peak": (C.c_int, [C.c_void_p, _dp]),
        "sf_measure_step_kernel": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _dp, _dp]),
        "sf_ctx_set_exchange": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _ALLGATHER_FN, C.c_void_p]),
        "sf_ctx_hint_next_seed": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int]),
        "sf_mt_jump_poly": (C.c_int, [C.c_uint64, _u64p]),
        "sf_ctx_set_l2_flush": (C.c_int, [C.c_void_p, C.c_uint64]),
        "sf_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "sf_ctx_init_comm": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int, C.c_int]),
        "sf_plan_frame_sharded": (C.c_int, [C.c_void_p, W, _dp, _dp, P, C.c_uint64, _dp, _u32p,
                                            C.c_uint32, Pr, _dp, _u64p]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("SEPSO_LIB") and not hasattr(L, name):
            continue            # an older experiment build (A/B timing): bind what it has
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _LIB = L
    return L


def _hyper_rows(hypers, groups, where):
    """The C ABI reads exactly `groups` rows; a mismatch is the reference's
    "hyper matrix group count != G" (swarm.hpp:101-102, planner.hpp:87-88)."""
    h = np.ascontiguousarray(hypers, dtype=np.float64)
    if h.ndim != 2 or h.shape[1] != 6 or h.shape[0] != groups:
        raise ValueError(f"{where}: hyper matrix group count != G")
    return h


def _check(status, bad=None):
    if status == SF_OK:
        return
    msg = (lib().sf_last_error() or b"").decode()
    if status == SF_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == SF_NON_FINITE:
        b = list(bad) if bad is not None else [0, 0, 0]
        raise NonFiniteFitnessError(b[0], b[1], b[2], msg)
    if status == SF_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == SF_RUNTIME_ERROR:
        raise RuntimeError(msg)
    raise CudaError(msg)


# ------------------------------------------------------------- value types
DEFAULT_GROUP_HYPERS = np.array([   # hypers.hpp:51-63 (PAPER Table 8)
    [2, 1, 1, 0.4, 0.2, 0.2], [1, 1, 2, 0.7, 0.3, 0.1], [2, 2, 1, 0.8, 0.1, 0.6],
    [2, 2, 1, 0.8, 0.6, 0.4], [2, 1, 2, 0.2, 0.1, 0.3], [2, 1, 2, 0.9, 0.5, 0.5],
    [1, 2, 2, 0.4, 0.1, 0.8], [1, 2, 2, 0.9, 0.3, 0.3]], dtype=np.float64)
EVOLVED_PATH_HYPERS = np.array([    # hypers.hpp:75-87 (PAPER Table 10)
    [1.53, 1.29, 1.34, 0.48, 0.19, 0.35], [1.72, 1.53, 1.34, 0.73, 0.28, 0.32],
    [1.34, 1.42, 1.33, 0.48, 0.21, 0.62], [1.76, 1.60, 1.21, 0.47, 0.30, 0.63],
    [1.68, 1.27, 1.25, 0.73, 0.36, 0.41], [1.66, 1.54, 1.54, 0.39, 0.16, 0.45],
    [1.57, 1.48, 1.75, 0.56, 0.34, 0.38], [1.31, 1.71, 1.23, 0.36, 0.25, 0.50]],
    dtype=np.float64)


def default_group_hypers():
    return DEFAULT_GROUP_HYPERS.copy()


def evolved_path_hypers():
    return EVOLVED_PATH_HYPERS.copy()


@dataclasses.dataclass
class PlannerConfig:
    """planner.hpp:19-57."""
    alpha: float = 30.0
    beta: float = 4.0
    gamma: float = 0.25
    delta: float = 10.0
    tw: int = 20
    pi_radius: float = 20.0
    max_iters_per_frame: int = 50
    groups: int = 8
    per_group: int = 170
    dim: int = 16
    auto_truncate: bool = True
    window_carryover: bool = False

    def waypoints(self):
        return self.dim // 2

    def pi_count(self):
        return int(self.gamma * float(self.per_group))

    def _c(self):
        return _PlannerCfg(self.alpha, self.beta, self.gamma, self.delta, self.tw, self.pi_radius,
                           self.max_iters_per_frame, self.groups, self.per_group, self.dim,
                           int(self.auto_truncate), int(self.window_carryover))


@dataclasses.dataclass
class ScenarioConfig:
    """simenv.hpp:17-40."""
    map_size: float = 366.0
    dynamic_obstacles: int = 6
    static_obstacles: int = 2
    min_side: float = 30.0
    max_side: float = 80.0
    max_speed: float = 5.0
    start_speed: float = 3.0
    target_speed: float = 8.0
    frames: int = 100
    dt: float = 1.0
    root_seed: int = 1

    def _c(self):
        return _ScenarioCfg(self.map_size, self.dynamic_obstacles, self.static_obstacles,
                            self.min_side, self.max_side, self.max_speed, self.start_speed,
                            self.target_speed, self.frames, self.dt, self.root_seed)


@dataclasses.dataclass
class PlanRecord:
    """planner.hpp:60-70 (best_path as an (W, 2) array of waypoints)."""
    best_path: np.ndarray
    fitness: float
    length: float
    intersections: int
    iterations: int
    truncated: bool
    stop_reason: str
    collision_free: bool
    wall_seconds: float

    @staticmethod
    def _from(rec: _PlanRecord, best: np.ndarray) -> "PlanRecord":
        W = best.size // 2
        return PlanRecord(np.stack([best[:W], best[W:]], axis=1), rec.fitness, rec.length,
                          int(rec.intersections), int(rec.iterations), bool(rec.truncated),
                          "converged" if rec.truncated else "cap", bool(rec.collision_free),
                          rec.wall_seconds)


class PolygonWorld:
    """geometry.hpp:42-67: map size, moving endpoints, closed polygon obstacles."""

    def __init__(self, width, height, start, target, obstacles: Sequence = (),
                 start_velocity=(0.0, 0.0), target_velocity=(0.0, 0.0), velocities=None):
        self.width, self.height = float(width), float(height)
        self.start = np.array(start, dtype=np.float64)
        self.target = np.array(target, dtype=np.float64)
        self.start_velocity = np.array(start_velocity, dtype=np.float64)
        self.target_velocity = np.array(target_velocity, dtype=np.float64)
        polys = [np.asarray(p, dtype=np.float64).reshape(-1, 2) for p in obstacles]
        self.offsets = np.zeros(len(polys) + 1, dtype=np.uint32)
        for i, p in enumerate(polys):
            self.offsets[i + 1] = self.offsets[i] + len(p)
        self.vertices = (np.ascontiguousarray(np.concatenate(polys)) if polys
                         else np.zeros((1, 2), dtype=np.float64))
        self.velocities = (np.asarray(velocities, dtype=np.float64).reshape(-1, 2).copy()
                           if velocities is not None else np.zeros((max(len(polys), 1), 2)))

    @property
    def n_obstacles(self):
        return len(self.offsets) - 1

    def obstacles(self):
        return [self.vertices[self.offsets[i]:self.offsets[i + 1]] for i in range(self.n_obstacles)]

    def copy(self):
        return PolygonWorld(self.width, self.height, self.start, self.target, self.obstacles(),
                            self.start_velocity, self.target_velocity, self.velocities.copy())

    def _c(self) -> _World:
        P = C.POINTER(_Point)
        return _World(self.width, self.height, _Point(*self.start), _Point(*self.target),
                      _Point(*self.start_velocity), _Point(*self.target_velocity),
                      self.n_obstacles, self.offsets.ctypes.data_as(_u32p),
                      self.vertices.ctypes.data_as(P), self.velocities.ctypes.data_as(P))

    def _absorb(self, w: _World):
        self.start = np.array([w.start.x, w.start.y])
        self.target = np.array([w.target.x, w.target.y])
        self.start_velocity = np.array([w.start_velocity.x, w.start_velocity.y])
        self.target_velocity = np.array([w.target_velocity.x, w.target_velocity.y])


def encode_path(waypoints) -> np.ndarray:
    """geometry.hpp:86-94: (W, 2) waypoints -> [x_1..x_W, y_1..y_W]."""
    w = np.asarray(waypoints, dtype=np.float64).reshape(-1, 2)
    return np.concatenate([w[:, 0], w[:, 1]])


def derive_seed(root: int, tag: str, index: Optional[int] = None) -> int:
    """rng.hpp:52-59 (named sub-stream seeds), computed by the engine library."""
    t = tag.encode()
    return int(lib().sf_derive_seed(root, t, len(t), 0 if index is None else 1, 0 if index is None else index))


def generate_world(config: ScenarioConfig, seed: int, rng: str = "mt19937") -> PolygonWorld:
    """simenv.hpp:83-132 on the host, drawing the given stream."""
    n = config.dynamic_obstacles + config.static_obstacles
    off = np.zeros(n + 1, dtype=np.uint32)
    verts = np.zeros((4 * n, 2))
    vel = np.zeros((max(n, 1), 2))
    w = _World()
    P = C.POINTER(_Point)
    _check(lib().sf_generate_world(C.byref(config._c()), seed, RNGS[rng], C.byref(w), _p(off, _u32p),
                                   verts.ctypes.data_as(P), vel.ctypes.data_as(P)))
    out = PolygonWorld(w.width, w.height, (w.start.x, w.start.y), (w.target.x, w.target.y),
                       [verts[4 * i:4 * i + 4] for i in range(n)],
                       (w.start_velocity.x, w.start_velocity.y),
                       (w.target_velocity.x, w.target_velocity.y), vel[:n] if n else None)
    return out


def step_world(world: PolygonWorld, dt: float) -> PolygonWorld:
    """simenv.hpp:155-184 (returns the advanced copy)."""
    nxt = world.copy()
    w = nxt._c()
    P = C.POINTER(_Point)
    _check(lib().sf_step_world(C.byref(w), nxt.vertices.ctypes.data_as(P),
                               nxt.velocities.ctypes.data_as(P), dt))
    nxt._absorb(w)
    return nxt


def should_truncate(window, best_is_collision_free: bool, config: PlannerConfig) -> bool:
    """planner.hpp:138-149."""
    w = np.ascontiguousarray(window, dtype=np.float64)
    r = C.c_int(0)
    _check(lib().sf_should_truncate(_p(w), len(w), int(best_is_collision_free),
                                    C.byref(config._c()), C.byref(r)))
    return bool(r.value)


# --------------------------------------------------------------- the engine
class Engine:
    """One device context (stream + device arena); fp32 = production, fp64 = parity."""

    def __init__(self, device: int = 0, precision: str = "fp32", rng: str = "mt19937"):
        self._L = lib()
        self.precision = FP64 if precision == "fp64" else FP32
        h = C.c_void_p()
        _check(self._L.sf_ctx_create(device, self.precision, C.byref(h)))
        self._h = h
        self.rng = rng
        _check(self._L.sf_ctx_set_rng(self._h, RNGS[rng]))

    def close(self):
        if getattr(self, "_h", None):
            self._L.sf_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    @property
    def stream(self) -> int:
        return self._L.sf_ctx_stream(self._h) or 0

    def synchronize(self):
        _check(self._L.sf_ctx_synchronize(self._h))

    def set_launch(self, cluster=0, threads=0):
        _check(self._L.sf_ctx_set_launch(self._h, cluster, threads))

    def enable_timing(self, on=True):
        _check(self._L.sf_ctx_enable_timing(self._h, int(on)))

    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().sf_comm_unique_id(buf))
        return bytes(buf)

    def init_comm(self, uid: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128)(*uid)
        _check(self._L.sf_ctx_init_comm(self._h, buf, nranks, rank))

    def set_exchange(self, nranks: int, rank: int, allgather=None):
        """Shard plan_frame_sharded / evolve over a host all-gather instead of
        NCCL: allgather(bytes) -> every rank's bytes concatenated in rank order
        (e.g. a gloo process group).  set_exchange(1, 0) resets."""
        if allgather is None:
            fn = _ALLGATHER_FN()
        else:
            def cb(user, send, recv, nbytes):
                try:
                    out = allgather(C.string_at(send, nbytes))
                    if len(out) != nbytes * nranks:
                        return 1
                    C.memmove(recv, out, len(out))
                    return 0
                except Exception:
                    return 1
            fn = _ALLGATHER_FN(cb)
        self._xfn = fn                     # the library keeps the pointer: keep the callback alive
        _check(self._L.sf_ctx_set_exchange(self._h, nranks, rank, fn, None))

    def plan_frame_sharded(self, world: PolygonWorld, prev_best, hypers, config: PlannerConfig,
                           seed: int, carried_window: Optional[list] = None):
        """plan_frame for one large swarm split by group over the communicator."""
        hyp = _hyper_rows(hypers, config.groups, "priori_init")
        prev = None if prev_best is None else np.ascontiguousarray(
            encode_path(prev_best) if np.ndim(prev_best) == 2 else prev_best, dtype=np.float64)
        best = np.zeros(config.dim)
        rec = _PlanRecord()
        bad = (C.c_uint64 * 3)()
        win = wl = None
        cap = 0
        if carried_window is not None:
            cap = max(len(carried_window), config.tw) + 1
            win = np.zeros(cap)
            win[:len(carried_window)] = carried_window
            wl = C.c_uint32(len(carried_window))
        st = self._L.sf_plan_frame_sharded(self._h, C.byref(world._c()), _p(prev), _p(hyp),
                                           C.byref(config._c()), C.c_uint64(seed), _p(win),
                                           C.byref(wl) if wl is not None else None, cap,
                                           C.byref(rec), _p(best), bad)
        _check(st, bad)
        if carried_window is not None and config.window_carryover:
            carried_window[:] = list(win[:wl.value])
        return PlanRecord._from(rec, best)

    def set_l2_flush(self, nbytes: int):
        _check(self._L.sf_ctx_set_l2_flush(self._h, nbytes))

    def measure_fp32_peak(self):
        t = C.c_double(0)
        _check(self._L.sf_measure_fp32_peak(self._h, C.byref(t)))
        return t.value

    def measure_step_kernel(self, groups, per_group, dim, reps=5):
        """K1 alone on a synthetic FP32 swarm: (ms per launch, algorithmic bytes per launch)."""
        ms, by = C.c_double(0), C.c_double(0)
        _check(self._L.sf_measure_step_kernel(self._h, groups, per_group, dim, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def last_io_bytes(self):
        a, b = C.c_uint64(0), C.c_uint64(0)
        _check(self._L.sf_ctx_last_io_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def kernel_time(self):
        ms, n = C.c_double(0), C.c_uint64(0)
        _check(self._L.sf_ctx_kernel_time(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    # -- planner.hpp:156-199
    def hint_next_seed(self, seed: Optional[int]):
        """The seed of the frame after the next plan_frame call (None clears):
        that call starts the next frame's init walk while it plans."""
        _check(self._L.sf_ctx_hint_next_seed(self._h, C.c_uint64(seed or 0), 0 if seed is None else 1))

    def plan_frame(self, world: PolygonWorld, prev_best, hypers, config: PlannerConfig,
                   seed: int, carried_window: Optional[list] = None):
        """Returns a PlanRecord; `carried_window` (a list) is updated in place."""
        hyp = _hyper_rows(hypers, config.groups, "priori_init")
        prev = None if prev_best is None else np.ascontiguousarray(
            encode_path(prev_best) if np.ndim(prev_best) == 2 else prev_best, dtype=np.float64)
        best = np.zeros(config.dim)
        rec = _PlanRecord()
        bad = (C.c_uint64 * 3)()
        win = wl = None
        cap = 0
        if carried_window is not None:
            cap = max(len(carried_window), config.tw) + 1
            win = np.zeros(cap)
            win[:len(carried_window)] = carried_window
            wl = C.c_uint32(len(carried_window))
        st = self._L.sf_plan_frame(self._h, C.byref(world._c()), _p(prev), _p(hyp),
                                   C.byref(config._c()), C.c_uint64(seed), _p(win),
                                   C.byref(wl) if wl is not None else None, cap, C.byref(rec),
                                   _p(best), bad)
        _check(st, bad)
        if carried_window is not None and config.window_carryover:
            carried_window[:] = list(win[:wl.value])
        return PlanRecord._from(rec, best)

    def plan_frames_batched(self, worlds: Sequence[PolygonWorld], prev, has_prev, hypers,
                            config: PlannerConfig, seeds, windows=None, window_lens=None):
        n = len(worlds)
        cw = (_World * n)(*[w._c() for w in worlds])
        hyp = _hyper_rows(hypers, config.groups, "priori_init")
        prev_a = None if prev is None else np.ascontiguousarray(prev, dtype=np.float64)
        hp = None if has_prev is None else np.ascontiguousarray(has_prev, dtype=np.uint8)
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        recs = (_PlanRecord * n)()
        best = np.zeros((n, config.dim))
        stat = np.zeros(n, dtype=np.int32)
        bad = np.zeros(3 * n, dtype=np.uint64)
        st = self._L.sf_plan_frames_batched(self._h, n, cw, _p(prev_a), _p(hp, _u8p), _p(hyp),
                                            C.byref(config._c()), _p(sd, _u64p), _p(windows),
                                            _p(window_lens, _u32p), recs, _p(best),
                                            _p(stat, _i32p), _p(bad, _u64p))
        _check(st)
        return [PlanRecord._from(recs[i], best[i]) for i in range(n)], best, stat

    # -- problems
    def _problem(self, problem, dim=None, lo=None, hi=None, world=None, alpha=30.0, beta=4.0):
        kind = PROBLEMS[problem] if isinstance(problem, str) else int(problem)
        keep = {}
        if kind == 0:
            cw = world._c()
            keep["w"] = cw
            pr = _Problem(0, dim, None, None, C.pointer(cw), alpha, beta)
        else:
            lo = np.full(dim, -600.0) if lo is None else np.ascontiguousarray(lo, dtype=np.float64)
            hi = np.full(dim, 600.0) if hi is None else np.ascontiguousarray(hi, dtype=np.float64)
            keep["lo"], keep["hi"] = lo, hi
            pr = _Problem(kind, dim, _p(lo), _p(hi), None, alpha, beta)
        keep["pr"] = pr
        return pr, keep

    # -- runner.hpp:97-129
    def run_dtpso(self, problem, hypers, groups, per_group, iterations, seed, dim=30, **kw):
        pr, keep = self._problem(problem, dim, **kw)
        hyp = _hyper_rows(hypers, groups, "init_swarm")
        trace = np.zeros(iterations)
        fp = np.zeros(dim)
        ff = C.c_double(0)
        bad = (C.c_uint64 * 3)()
        st = self._L.sf_run_dtpso(self._h, C.byref(pr), _p(hyp), groups, per_group, iterations,
                                  C.c_uint64(seed), _p(trace), _p(fp), C.byref(ff), bad)
        _check(st, bad)
        return dict(trace=trace, final_point=fp, final_fitness=ff.value,
                    evaluations=groups * per_group * iterations)

    def run_dtpso_batched(self, problem, hypers, groups, per_group, iterations, seeds, dim=30,
                          per_run_hypers=False, **kw):
        pr, keep = self._problem(problem, dim, **kw)
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        n = len(sd)
        hyp = np.ascontiguousarray(hypers, dtype=np.float64)
        traces = np.zeros((n, iterations))
        fps = np.zeros((n, dim))
        ffs = np.zeros(n)
        stat = np.zeros(n, dtype=np.int32)
        _check(self._L.sf_run_dtpso_batched(self._h, C.byref(pr), n, _p(hyp), int(per_run_hypers),
                                            groups, per_group, iterations, _p(sd, _u64p),
                                            _p(traces), _p(fps), _p(ffs), _p(stat, _i32p)))
        return traces, fps, ffs, stat

    # -- hsef.hpp
    def lfv_batch(self, problem, candidates, seeds, inner_groups, inner_per_group,
                  inner_iterations, dim=30, **kw):
        pr, keep = self._problem(problem, dim, **kw)
        cand = np.ascontiguousarray(candidates, dtype=np.float64)
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        out = np.zeros(len(sd))
        _check(self._L.sf_lfv_batch(self._h, C.byref(pr), len(sd), _p(cand), _p(sd, _u64p),
                                    inner_groups, inner_per_group, inner_iterations, _p(out)))
        return out

    def lfv_fitness(self, candidate, problem, inner_groups, inner_per_group, inner_iterations,
                    seed, dim=30, **kw):
        return float(self.lfv_batch(problem, np.asarray(candidate)[None], [seed], inner_groups,
                                    inner_per_group, inner_iterations, dim, **kw)[0])

    def evolve(self, problem, inner, outer, seed, outer_hypers=None, dim=30, **kw):
        """inner = (G, N, T); outer = (G, N, E).  hsef.hpp:125-171."""
        pr, keep = self._problem(problem, dim, **kw)
        oh = np.ascontiguousarray(DEFAULT_GROUP_HYPERS if outer_hypers is None else outer_hypers,
                                  dtype=np.float64)
        E = outer[2]
        bt, rt = np.zeros(E), np.zeros(E)
        best = np.zeros(6 * inner[0])
        _check(self._L.sf_evolve(self._h, C.byref(pr), inner[0], inner[1], inner[2], outer[0],
                                 outer[1], E, C.c_uint64(seed), _p(oh), _p(bt), _p(rt), _p(best),
                                 None, None))
        return dict(best_lfv_trace=bt, evolution_lfv_trace=rt, best=best.reshape(-1, 6),
                    evolutions=E, lfv_evaluations=outer[0] * outer[1] * E)

    # -- stages
    def init_swarm(self, hypers, lo, hi, G, N, D, seed, prev=None, warm=0, pi_radius=20.0,
                   first_draw=0):
        x = np.zeros(G * N * D)
        v = np.zeros(G * N * D)
        hyp = np.ascontiguousarray(hypers, dtype=np.float64)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        pv = None if prev is None else np.ascontiguousarray(prev, dtype=np.float64)
        _check(self._L.sf_init_swarm(self._h, _p(hyp), _p(lo), _p(hi), G, N, D, C.c_uint64(seed),
                                     C.c_uint64(first_draw), _p(pv), warm, pi_radius, _p(x), _p(v)))
        return x, v

    def step(self, hypers, lo, hi, G, N, D, x, v, pbest_x, gbest_x, tbest_x, seed, first_draw,
             k, T):
        x = np.array(x, dtype=np.float64)
        v = np.array(v, dtype=np.float64)
        arr = [np.ascontiguousarray(a, dtype=np.float64) for a in (hypers, lo, hi, pbest_x, gbest_x, tbest_x)]
        _check(self._L.sf_step(self._h, _p(arr[0]), _p(arr[1]), _p(arr[2]), G, N, D, _p(x), _p(v),
                               _p(arr[3]), _p(arr[4]), _p(arr[5]), C.c_uint64(seed),
                               C.c_uint64(first_draw), k, T))
        return x, v

    def update_bests(self, G, N, D, x, pbx, pbf, gbx, gbf, tbx, tbf, fitness):
        pbx, pbf, gbx, gbf, tbx = (np.array(a, dtype=np.float64) for a in (pbx, pbf, gbx, gbf, tbx))
        t = C.c_double(tbf)
        xa = np.ascontiguousarray(x, dtype=np.float64)
        fa = np.ascontiguousarray(fitness, dtype=np.float64)
        _check(self._L.sf_update_bests(self._h, G, N, D, _p(xa), _p(pbx), _p(pbf), _p(gbx),
                                       _p(gbf), _p(tbx), C.byref(t), _p(fa)))
        return pbx, pbf, gbx, gbf, tbx, t.value

    def eval_path_rows(self, world: PolygonWorld, xs, dim, alpha=30.0, beta=4.0):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        rows = xs.size // dim
        f = np.zeros(rows)
        q = np.zeros(rows, dtype=np.uint32)
        _check(self._L.sf_eval_path_rows(self._h, C.byref(world._c()), _p(xs), rows, dim, alpha,
                                         beta, _p(f), _p(q, _u32p)))
        return f, q

    def eval_bench_rows(self, problem, xs, dim):
        kind = PROBLEMS[problem] if isinstance(problem, str) else int(problem)
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        rows = xs.size // dim
        f = np.zeros(rows)
        _check(self._L.sf_eval_bench_rows(self._h, kind, _p(xs), rows, dim, _p(f)))
        return f

    # -- simenv.hpp:239-276
    def run_scenario(self, config: ScenarioConfig, variant: str, frames: int,
                     base: Optional[PlannerConfig] = None, evolved=None):
        base = base or PlannerConfig()
        ev = np.ascontiguousarray(EVOLVED_PATH_HYPERS if evolved is None else evolved,
                                  dtype=np.float64)
        recs = (_PlanRecord * frames)()
        dim = base.dim
        best = np.zeros((frames, dim))
        if ev.size % 6 != 0:
            raise ValueError("HyperMatrix: rows of 6 values required")
        _check(self._L.sf_run_scenario(self._h, C.byref(config._c()), VARIANTS.index(variant),
                                       frames, C.byref(base._c()), _p(ev), ev.size // 6, recs, _p(best)))
        return [PlanRecord._from(recs[i], best[i]) for i in range(frames)]


class SceneBatch:
    """Device-resident run_scenario for n scenarios (sf_scene_batch_*): each
    frame is one fused planning launch + one on-device step_world launch."""

    def __init__(self, engine: Engine, scenarios: Sequence[ScenarioConfig],
                 planner: PlannerConfig, hypers, max_frames: int):
        self._e = engine
        self.n = len(scenarios)
        self.dim = planner.dim
        cfgs = (_ScenarioCfg * self.n)(*[s._c() for s in scenarios])
        hyp = _hyper_rows(hypers, planner.groups, "priori_init")
        h = C.c_void_p()
        _check(engine._L.sf_scene_batch_create(engine._h, self.n, cfgs, C.byref(planner._c()),
                                               _p(hyp), max_frames, C.byref(h)))
        self._h = h

    def run(self, frames: int):
        _check(self._e._L.sf_scene_batch_run(self._h, frames))

    def records(self, first: int, count: int, with_best: bool = False):
        recs = (_PlanRecord * (count * self.n))()
        best = np.zeros((count, self.n, self.dim)) if with_best else None
        _check(self._e._L.sf_scene_batch_records(self._h, first, count, recs, _p(best)))
        out = [PlanRecord._from(recs[i], best.reshape(-1, self.dim)[i] if with_best
                                else np.zeros(self.dim)) for i in range(count * self.n)]
        return out, best

    def close(self):
        if getattr(self, "_h", None):
            self._e._L.sf_scene_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
