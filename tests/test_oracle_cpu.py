"""Pin the CPU oracle (oracle/liboracle.so) to the reference -- CPU only.

(a) golden vectors produced by the reference itself (tests/golden/
    reference_vectors.json, from tests/golden/make_golden.py over oracle/_ref);
(b) the reference's own known-answer constants (test_rng.cpp, test_geometry.cpp,
    test_benchmarks.cpp, test_hsef.cpp, proj/test_output.txt);
(c) live comparisons against oracle/_ref when it is built (build container).
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle_lib import ROOT
from oracle_lib import (DEFAULT_GROUP_HYPERS, EVOLVED_PATH_HYPERS, RNG_MT, RNG_PHILOX, WorldBuf,
                        generate_world, oracle, oracle_plan_frame, oracle_run_dtpso, planner_cfg,
                        ptr, rect, ref, ref_plan_frame, u32p)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


def stream(kind, seed, n):
    o = oracle()
    if kind == "philox":
        return [(o.or_philox_word(seed, i) >> 11) * 2.0 ** -53 for i in range(n)]
    # mt19937_64 stream through the plan-frame-free path: first n words
    out = []
    for i in range(1, n + 1):
        out.append((o.or_mt_nth(seed, i) >> 11) * 2.0 ** -53)
    return out


# ------------------------------------------------------------------- rng.hpp
def test_mt19937_10000th_output():
    """test_rng.cpp:35-41: the standard fixes the 10000th default-seeded output."""
    assert oracle().or_mt_nth(5489, 10000) == 9981545732273789042


def test_philox_known_answers():
    """Philox4x32-10 known-answer vectors (Random123 kat_vectors)."""
    o = oracle()
    out = (C.c_uint32 * 4)()
    kats = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
            ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
            ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
             (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]
    for ctr, key, want in kats:
        o.or_philox4x32_10((C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), out)
        assert tuple(out) == want


@pytest.mark.parametrize("kind", ["mt", "philox"])
def test_uniform_streams_match_reference(kind):
    for seed, vals in GOLD["rng"][kind].items():
        assert stream(kind, int(seed), 8) == vals


def test_derive_seed_matches_reference():
    o = oracle()
    for r, t, v in GOLD["rng"]["derive_seed"]:
        assert o.or_derive_seed(r, t.encode()) == v
    for r, t, i, v in GOLD["rng"]["derive_seed_idx"]:
        assert o.or_derive_seed_idx(r, t.encode(), i) == v


# -------------------------------------------------------------- geometry.hpp
def test_segment_corpus_matches_reference():
    """acceptance.cpp:390-407 corpus + 300 integer-grid pairs (exact predicates)."""
    o = oracle()
    for a1, a2, b1, b2, want in GOLD["segments"]:
        arr = [np.array(p, dtype=np.float64) for p in (a1, a2, b1, b2)]
        assert o.or_segments_intersect(*(ptr(x) for x in arr)) == want


def test_exact_integer_oracle_on_grid_pairs():
    """test_geometry.cpp:122-143: agrees with an exact integer predicate."""
    o = oracle()
    g = np.random.default_rng(90210)

    def orient(a, b, c):
        v = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
        return (v > 0) - (v < 0)

    def on_seg(a, b, p):
        return min(a[0], b[0]) <= p[0] <= max(a[0], b[0]) and min(a[1], b[1]) <= p[1] <= max(a[1], b[1])

    def exact(a1, a2, b1, b2):
        o1, o2, o3, o4 = orient(a1, a2, b1), orient(a1, a2, b2), orient(b1, b2, a1), orient(b1, b2, a2)
        return ((o1 != o2 and o3 != o4) or (o1 == 0 and on_seg(a1, a2, b1)) or (o2 == 0 and on_seg(a1, a2, b2))
                or (o3 == 0 and on_seg(b1, b2, a1)) or (o4 == 0 and on_seg(b1, b2, a2)))

    hits = 0
    for trial in range(6000):
        r = 4 if trial % 3 == 0 else 40
        pts = [tuple(int(v) for v in g.integers(-r, r + 1, 2)) for _ in range(4)]
        got = o.or_segments_intersect(*(ptr(np.array(p, dtype=np.float64)) for p in pts))
        assert got == exact(*pts)
        hits += got
    assert hits > 300


def test_point_strictly_inside_matches_reference():
    o = oracle()
    for poly, p, want in GOLD["inside"]:
        pa, pp = np.array(poly, dtype=np.float64), np.array(p, dtype=np.float64)
        assert o.or_point_strictly_inside(ptr(pp), ptr(pa), len(poly) // 2) == want


def test_grid_world_fitness_matches_reference():
    o = oracle()
    for case in GOLD["grid_worlds"]:
        w = WorldBuf(40.0, 40.0, case["start"], case["target"], case["obstacles"])
        xs = np.array(case["xs"], dtype=np.float64)
        f, q = np.zeros(len(xs)), np.zeros(len(xs), dtype=np.uint32)
        o.or_eval_path_rows(ptr(xs), len(xs), case["D"], C.byref(w.struct()), 30.0, 4.0, ptr(f), ptr(q, u32p))
        assert q.tolist() == case["q"]
        assert f.tolist() == case["fitness"]


def test_paper_paths_match_reference():
    o = oracle()
    pp = GOLD["paper_paths"]
    w = WorldBuf.__new__(WorldBuf)
    w.head, w.offsets = np.array(pp["head"]), np.array(pp["offsets"], dtype=np.uint32)
    w.verts, w.vel, w.n = np.array(pp["verts"]), np.array(pp["vel"]), len(pp["offsets"]) - 1
    xs = np.array(pp["xs"])
    f, q = np.zeros(len(xs)), np.zeros(len(xs), dtype=np.uint32)
    o.or_eval_path_rows(ptr(xs), len(xs), 16, C.byref(w.struct()), 30.0, 4.0, ptr(f), ptr(q, u32p))
    assert q.tolist() == pp["q"] and f.tolist() == pp["fitness"]


def test_fixture_q4_and_penalty():
    """test_geometry.cpp:158-171 and 288-296."""
    o = oracle()
    w = WorldBuf(10.0, 10.0, (0.0, 3.0), (0.0, 6.0), [rect(2, 2, 6, 6)])
    p = np.array([8.0, 0.0, 3.0, 5.0])
    assert o.or_count_intersections(ptr(p), 4, C.byref(w.struct())) == 4
    assert abs(30.0 * 4.0 ** 4 - 7680.0) == 0


def test_glibc_hypot_restatement():
    """The FP64 engine's hypot (geometry.cuh:hypot_glibc, Borges' corrected
    kernel without FMA) equals libm's std::hypot bit for bit."""
    g = np.random.default_rng(7)
    x = g.uniform(-500, 500, 400000)
    y = g.uniform(-500, 500, 400000)
    x[::4] = np.floor(x[::4])
    y[::7] = x[::7] * (1 + 1e-9 * g.uniform(0, 1, len(y[::7])))
    ax, ay = np.maximum(np.abs(x), np.abs(y)), np.minimum(np.abs(x), np.abs(y))
    with np.errstate(all="ignore"):
        h = np.sqrt(ax * ax + ay * ay)
        small = h <= 2.0 * ay
        d1 = h - ay
        t1a = ax * (2.0 * d1 - ax)
        t2a = (d1 - 2.0 * (ax - ay)) * d1
        d2 = h - ax
        t1b = 2.0 * d2 * (ax - 2.0 * ay)
        t2b = (4.0 * d2 - ay) * ay + d2 * d2
        t1 = np.where(small, t1a, t1b)
        t2 = np.where(small, t2a, t2b)
        r = h - (t1 + t2) / (2.0 * h)
    r = np.where(ay <= ax * 2.0 ** -54, ax + ay, r)
    assert np.array_equal(r, np.hypot(x, y))


# ----------------------------------------------------------- benchmarks.hpp
def test_benchmarks_match_reference():
    o = oracle()
    for case in GOLD["bench"]:
        for row, want in zip(case["xs"], case["f"]):
            assert o.or_bench_eval(case["kind"], ptr(np.array(row)), case["D"]) == want


def test_benchmark_spot_values():
    """test_benchmarks.cpp:82-93."""
    o = oracle()
    assert o.or_bench_eval(1, ptr(np.array([1.0, 2.0, 3.0])), 3) == 14.0
    assert o.or_bench_eval(2, ptr(np.zeros(2)), 2) == 1.0
    assert abs(o.or_bench_eval(3, ptr(np.full(4, 0.5)), 4) - 81.0) < 1e-12


# --------------------------------------------------------------- simenv.hpp
@pytest.mark.parametrize("kind", ["mt", "philox"])
def test_world_generation_and_stepping_match_reference(kind):
    o = oracle()
    sim = GOLD["simenv"][kind]
    w = generate_world("oracle", o.or_derive_seed(3, b"world"), RNG_MT if kind == "mt" else RNG_PHILOX)
    assert w.head.tolist() == sim["world"]["head"] and w.verts.tolist() == sim["world"]["verts"]
    assert w.vel.tolist() == sim["world"]["vel"]
    for _ in range(20):
        o.or_step_world(ptr(w.head), w.n, ptr(w.offsets, u32p), ptr(w.verts), ptr(w.vel), 1.0)
    assert w.head.tolist() == sim["after20"]["head"] and w.verts.tolist() == sim["after20"]["verts"]


# -------------------------------------------------------------- planner.hpp
@pytest.mark.parametrize("kind", ["mt", "philox"])
def test_plan_frames_match_reference(kind):
    o = oracle()
    rk = RNG_MT if kind == "mt" else RNG_PHILOX
    w = generate_world("oracle", o.or_derive_seed(3, b"world"), rk)
    cfg = planner_cfg(max_iters=30, window_carryover=1)
    prev, win = None, []
    for fr in GOLD["plan_frames"][kind]:
        st, rec, best, win, _ = oracle_plan_frame(w, prev, EVOLVED_PATH_HYPERS, cfg, fr["seed"], rk, win)
        assert st == 0
        assert (rec.fitness, rec.length, rec.intersections, rec.iterations, rec.truncated) == \
               (fr["fitness"], fr["length"], fr["q"], fr["iterations"], fr["truncated"])
        assert best.tolist() == fr["best"] and win.tolist() == fr["window"]
        prev = best
        o.or_step_world(ptr(w.head), w.n, ptr(w.offsets, u32p), ptr(w.verts), ptr(w.vel), 1.0)


def test_published_scenario_statistics():
    """proj/test_output.txt:25-27: seed 3, cap 30, carryover -> 16.2
    iterations/frame, 91/100 truncated, 0 colliding, 123.5 cm (mt stream)."""
    s = GOLD["scenario_seed3"]
    assert round(s["mean_iterations"], 1) == 16.2 and s["truncated"] == 91
    assert s["colliding_truncations"] == 0 and round(s["mean_length"], 1) == 123.5
    o = oracle()
    w = generate_world("oracle", o.or_derive_seed(3, b"world"), RNG_MT)
    cfg = planner_cfg(max_iters=30, window_carryover=1)
    prev, win, its = None, [], []
    for f in range(100):
        st, rec, best, win, _ = oracle_plan_frame(w, prev, EVOLVED_PATH_HYPERS, cfg,
                                                  o.or_derive_seed_idx(3, b"plan", f), RNG_MT, win)
        its.append(rec.iterations)
        prev = best
        o.or_step_world(ptr(w.head), w.n, ptr(w.offsets, u32p), ptr(w.verts), ptr(w.vel), 1.0)
    assert its == s["iterations"]


def test_truncation_rule_cases():
    """test_planner.cpp:80-118."""
    o = oracle()

    def st(window, cf, **kw):
        cfg = planner_cfg(tw=4, **kw)
        a = np.array(window, dtype=np.float64)
        return bool(o.or_should_truncate(ptr(a), len(a), int(cf), C.byref(cfg)))

    assert not st([5.0, 5.0, 5.0], True)
    assert st([42.0] * 4, True) and not st([42.0] * 4, False)
    assert not st([0, 100, 0, 100], True) and st([0, 100, 0, 100], True, delta=50.5)
    assert st([1, 2, 3, 4], True, delta=1.2) and not st([1, 2, 3, 4], True, delta=1.1)


# --------------------------------------------------------------- runner/hsef
def test_run_dtpso_matches_reference():
    for run in GOLD["run_dtpso_philox"]:
        st, tr, fp, ff, _ = oracle_run_dtpso(run["kind"], DEFAULT_GROUP_HYPERS, 8, 10, run["T"], run["seed"],
                                             D=30, lo=np.full(30, -600.0), hi=np.full(30, 600.0))
        assert st == 0 and tr.tolist() == run["trace"] and fp.tolist() == run["final_point"]


def test_unflatten_repair_matches_reference():
    """hsef.hpp:57-71 (test_hsef.cpp:106-126: clamp, swap after clamp)."""
    o = oracle()
    h = GOLD["hsef"]
    out = np.zeros(18)
    o.or_unflatten(ptr(np.array(h["raw"])), 3, ptr(out))
    assert out.tolist() == h["unflatten"]
    assert out[:6].tolist() == [2.5, 0.5, 0.5, 1.0, 0.05, 1.0]


def test_evolve_matches_reference():
    o = oracle()
    e = GOLD["hsef"]["evolve"]
    bt, rt, bh = np.zeros(3), np.zeros(3), np.zeros(24)
    lo, hi = np.full(6, -600.0), np.full(6, 600.0)
    st = o.or_evolve_flat(1, None, 6, ptr(lo), ptr(hi), 30.0, 4.0, 4, 5, 20, 2, 3, 3, e["seed"],
                          ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS[:2])), RNG_PHILOX,
                          ptr(bt), ptr(rt), ptr(bh))
    assert st == 0
    assert bt.tolist() == e["best_trace"] and rt.tolist() == e["round_trace"] and bh.tolist() == e["best"]


# ------------------------------------------------- live reference (optional)
needs_ref = pytest.mark.skipif(ref("philox") is None, reason="oracle/_ref not built")


@needs_ref
def test_live_batched_equals_reference_random_instances():
    """acceptance.cpp:73-113 style: 60 random (G, N, D, T) instances."""
    g = np.random.default_rng(20260815)
    for i in range(60):
        G, N, D, T = int(g.integers(1, 5)), int(g.integers(1, 9)), int(g.integers(1, 9)), int(g.integers(1, 21))
        kind = 1 + i % 4
        h = np.zeros((G, 6))
        h[:, :3] = g.uniform(0, 2.5, (G, 3))
        h[:, 4] = g.uniform(0.05, 0.5, G)
        h[:, 3] = h[:, 4] + g.uniform(0, 0.4, G)
        h[:, 5] = g.uniform(0.05, 1.0, G)
        for libk, rk in (("philox", RNG_PHILOX), ("mt", RNG_MT)):
            r = ref(libk)
            tr, fp, ff = np.zeros(T), np.zeros(D), C.c_double(0)
            bad = (C.c_size_t * 3)()
            assert r.ref_run_dtpso(kind, None, D, 30.0, 4.0, ptr(h), G, N, T, 1000 + i, ptr(tr), ptr(fp),
                                   C.byref(ff), bad) == 0
            st, tr2, fp2, ff2, _ = oracle_run_dtpso(kind, h, G, N, T, 1000 + i, D=D, lo=np.full(D, -600.0),
                                                    hi=np.full(D, 600.0), rng=rk)
            assert st == 0 and tr.tolist() == tr2.tolist() and fp.tolist() == fp2.tolist()


@needs_ref
def test_live_plan_frames_random_worlds():
    o = oracle()
    g = np.random.default_rng(5)
    for trial in range(6):
        w = generate_world("oracle", o.or_derive_seed(100 + trial, b"world"), RNG_PHILOX)
        cfg = planner_cfg(max_iters=int(g.integers(5, 25)), G=4, N=int(g.integers(5, 40)), D=2 * int(g.integers(1, 9)),
                          tw=int(g.integers(2, 8)), window_carryover=1, gamma=float(g.uniform(0, 1)))
        prev, win_o, win_r = None, [], []
        hyp = EVOLVED_PATH_HYPERS[:4]
        for f in range(4):
            seed = o.or_derive_seed_idx(100 + trial, b"plan", f)
            a = oracle_plan_frame(w, prev, hyp, cfg, seed, RNG_PHILOX, win_o)
            b = ref_plan_frame("philox", w, prev, hyp, cfg, seed, win_r)
            assert a[0] == b[0] == 0
            assert (a[1].fitness, a[1].iterations, a[1].truncated) == (b[1].fitness, b[1].iterations, b[1].truncated)
            assert a[2].tolist() == b[2].tolist() and a[3].tolist() == b[3].tolist()
            prev, win_o, win_r = a[2], a[3], b[3]


def test_glibc_cos_restatement(tmp_path):
    """The FP64 engine's cos (csrc/cos_glibc.cuh, the restated glibc 2.39 FMA
    build of s_sin.c), compiled for the host, equals libm's cos bit for bit on
    the benchmarks' argument distributions (2*pi*x and x/sqrt(i+1) over the
    box [-600, 600]) and on every branch of the algorithm."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    so = str(tmp_path / "libcoscheck.so")
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-shared", "-fPIC",
                    "-I" + os.path.join(ROOT, "paper_2308_10169_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "cos_check.cpp"), "-o", so], check=True)
    ours = C.CDLL(so)
    libm = C.CDLL("libm.so.6")
    libm.cos.restype, libm.cos.argtypes = C.c_double, [C.c_double]
    g = np.random.default_rng(21)
    n = 400_000
    p = g.uniform(-600, 600, n)
    xs = np.concatenate([2.0 * np.pi * p, p / np.sqrt(g.integers(1, 31, n)), g.uniform(-1, 1, n),
                         g.uniform(-3, 3, n), np.round(p) * 2 * np.pi, g.uniform(-1e5, 1e5, n),
                         g.uniform(-1e-7, 1e-7, 1000), [0.0, -0.0, 0.126, -0.126, 0.855469, 2.426265]])
    got = np.zeros_like(xs)
    ours.cos_glibc_rows(ptr(xs), len(xs), ptr(got))
    # libm through a vectorised ufunc would be numpy's own cos: call libm itself
    want = np.array([libm.cos(float(v)) for v in xs[::7]])
    assert np.array_equal(got[::7], want)


# ------------------------------------------- per-particle oracles (8(f) 4)
def test_scale_harness_batched_equals_per_particle():
    """The reference's `scale` check (proj/tools/swarmforge.cpp:202-255): the
    batched run_dtpso and the per-particle run_dppso_reference give identical
    traces from the same seed -- the wrapped oracle is the reference's own."""
    r = ref("mt")
    if r is None:
        pytest.skip("oracle/_ref not built")
    G, N, D, T = 8, 16, 8, 25
    h = np.ascontiguousarray(DEFAULT_GROUP_HYPERS)
    for kind in (1, 3):
        ta, fa, ffa = np.zeros(T), np.zeros(D), C.c_double(0)
        tb, fb, ffb, wall = np.zeros(T), np.zeros(D), C.c_double(0), C.c_double(0)
        bad = (C.c_size_t * 3)()
        assert r.ref_run_dtpso(kind, None, D, 30.0, 4.0, ptr(h), G, N, T, 77, ptr(ta), ptr(fa), C.byref(ffa), bad) == 0
        assert r.ref_run_dppso_reference(kind, None, D, 30.0, 4.0, ptr(h), G, N, T, 77, ptr(tb), ptr(fb),
                                         C.byref(ffb), C.byref(wall)) == 0
        assert np.array_equal(ta, tb) and np.array_equal(fa, fb) and ffa.value == ffb.value
        assert wall.value > 0.0
    # the classic PSO baseline runs and reports a non-increasing trace
    tp, fp, ffp, wall = np.zeros(T), np.zeros(D), C.c_double(0), C.c_double(0)
    assert r.ref_run_pso_reference(1, None, D, 30.0, 4.0, T, 40, 5, ptr(tp), ptr(fp), C.byref(ffp), C.byref(wall)) == 0
    assert np.all(np.diff(tp) <= 0) and ffp.value == tp[-1]
