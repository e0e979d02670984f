"""The C-ABI boundary, CPU only: the library loads, exports every entry point
declared in include/sepso.h, the ctypes mirror matches the C struct layouts,
and the host-side (CPU-owned) pieces behave like the reference."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2308_10169_b200 as pe
from paper_2308_10169_b200 import engine as E
from oracle_lib import RNG_PHILOX, generate_world, oracle, ptr, u32p

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sepso.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = pe.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(E.ABI_SYMBOLS) == syms
    assert lib.sf_abi_version() == 2


def test_library_is_sm100a_cuda():
    """The .so carries sm_100a SASS (no PTX-JIT fallback, no other arch)."""
    out = subprocess.run(["cuobjdump", "--list-elf", pe.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_struct_layouts_match_c():
    """sizeof/offsetof of the ABI structs seen by a C compiler == the ctypes mirror."""
    prog = r'''
#include <stddef.h>
#include <stdio.h>
#include "sepso.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(sf_world), sizeof(sf_planner_config),
         sizeof(sf_plan_record), sizeof(sf_problem), sizeof(sf_scenario_config), sizeof(sf_point));
  printf("%zu %zu %zu %zu\n", offsetof(sf_world, n_obstacles), offsetof(sf_planner_config, tw),
         offsetof(sf_plan_record, wall_seconds), offsetof(sf_scenario_config, root_seed));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        sizes, offs = subprocess.run([exe], capture_output=True, text=True).stdout.split("\n")[:2]
    assert [int(v) for v in sizes.split()] == [C.sizeof(t) for t in (
        E._World, E._PlannerCfg, E._PlanRecord, E._Problem, E._ScenarioCfg, E._Point)]
    assert [int(v) for v in offs.split()] == [E._World.n_obstacles.offset, E._PlannerCfg.tw.offset,
                                              E._PlanRecord.wall_seconds.offset,
                                              E._ScenarioCfg.root_seed.offset]


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(E, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(E, "_LIB", None)
    with pytest.raises(RuntimeError, match="not built"):
        E.lib()


def test_no_gpu_context_raises_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pe.CudaError):
        pe.Engine(0)


def test_should_truncate_host_predicate():
    """planner.hpp:138-149 via the C ABI (test_planner.cpp:80-118)."""
    c = pe.PlannerConfig(groups=2, per_group=8, dim=4, tw=4, max_iters_per_frame=12)
    assert not pe.should_truncate([5.0, 5.0, 5.0], True, c)
    assert pe.should_truncate([42.0] * 4, True, c)
    assert not pe.should_truncate([42.0] * 4, False, c)
    assert not pe.should_truncate([0.0, 100.0, 0.0, 100.0], True, c)
    c.delta = 50.5
    assert pe.should_truncate([0.0, 100.0, 0.0, 100.0], True, c)
    c.delta = 1.2
    assert pe.should_truncate([1.0, 2.0, 3.0, 4.0], True, c)
    c.delta = 1.1
    assert not pe.should_truncate([1.0, 2.0, 3.0, 4.0], True, c)
    c.tw, c.delta = 3, 10.0
    assert pe.should_truncate([1000.0, 5.0, 5.0, 5.0], True, c)


@pytest.mark.parametrize("rng,rk", [("mt19937", 0), ("philox", 1)])
def test_generate_and_step_world_match_oracle(rng, rk):
    """simenv.hpp:83-184 on the host, both streams == oracle, 50 steps."""
    o = oracle()
    for root in range(4):
        seed = o.or_derive_seed(root, b"world")
        w = pe.generate_world(pe.ScenarioConfig(), seed, rng)
        wo = generate_world("oracle", seed, rk)
        assert np.array_equal(w.vertices.reshape(-1), wo.verts)
        for _ in range(50):
            w = pe.step_world(w, 1.0)
            o.or_step_world(ptr(wo.head), wo.n, ptr(wo.offsets, u32p), ptr(wo.verts), ptr(wo.vel), 1.0)
        assert np.array_equal(w.vertices.reshape(-1), wo.verts)
        assert np.array_equal(w.start, wo.head[2:4]) and np.array_equal(w.target, wo.head[4:6])
        assert np.array_equal(w.velocities[:w.n_obstacles].reshape(-1), wo.vel)


def test_world_contract():
    """test_simenv.cpp:105-155: obstacles inside the map, clear of endpoints."""
    o = oracle()
    for root in range(20):
        w = pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(root, b"world"))
        assert w.n_obstacles == 8
        for poly in w.obstacles():
            assert np.all(poly >= 0) and np.all(poly <= 366.0)
            lo, hi = poly.min(0), poly.max(0)
            for p in (w.start, w.target):
                assert not (lo[0] - 2 <= p[0] <= hi[0] + 2 and lo[1] - 2 <= p[1] <= hi[1] + 2)
        sp = np.hypot(*w.velocities[:6].T)
        assert np.all((sp > 0) & (sp <= 5.0)) and np.all(w.velocities[6:] == 0)


def test_invalid_scenario_config_rejected():
    with pytest.raises(ValueError):
        pe.generate_world(pe.ScenarioConfig(max_side=400.0), 1)
    with pytest.raises(ValueError):
        pe.generate_world(pe.ScenarioConfig(max_speed=0.0), 1)


def test_dropin_headers_compile_as_cpp20():
    """A reference user's program compiles against include/swarmforge/*.hpp."""
    for ex in ("plan_route.cpp", "minimize_rastrigin.cpp"):
        subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", ex)], check=True)
