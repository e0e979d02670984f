"""B200-native SEPSO engine (arXiv 2308.10169) behind the reference planner API.

The compute path is ``lib/libsepso_cuda.so`` (sm_100a kernels + host C++ runtime,
C ABI in ``include/sepso.h``).  ``engine`` is a thin ctypes mirror of the
reference API for Python callers, tests and the benchmark.
"""
from .engine import (  # noqa: F401
    ABI_SYMBOLS, DEFAULT_GROUP_HYPERS, EVOLVED_PATH_HYPERS, CudaError, Engine,
    NonFiniteFitnessError, PlanRecord, SceneBatch, PlannerConfig, PolygonWorld, ScenarioConfig,
    default_group_hypers, derive_seed, encode_path, evolved_path_hypers, generate_world, lib,
    should_truncate, step_world, LIB_PATH,
)
