"""Jump-ahead for the reference's std::mt19937_64 stream (rng.hpp:13-28):
sf_mt_jump_poly(W) = x^W mod phi, and XOR-ing the raw windows x[i .. i+311]
over its terms gives the generator state W words later.  Checked here in numpy
against the plain recurrence; the device fill built on it is checked word for
word against the sequential fill in tests/test_gpu_mt.py."""
import ctypes as C
import time

import numpy as np
import pytest

import paper_2308_10169_b200 as pe

U64 = np.uint64
UPPER, LOWER = U64(0xFFFFFFFF80000000), U64(0x7FFFFFFF)
MAT = U64(0xB5026F5AA96619E9)


def seed_state(seed):
    x = [seed]
    for i in range(1, 312):
        p = x[-1]
        x.append((6364136223846793005 * (p ^ (p >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
    return np.array(x, dtype=U64)


def twist(a, b, m):
    y = (a & UPPER) | (b & LOWER)
    return m ^ (y >> U64(1)) ^ np.where((b & U64(1)) != 0, MAT, U64(0))


def raw(state, n):
    """state (312 raw words x[0..311]) followed by the next n raw words."""
    x = np.zeros(312 + ((n + 311) // 312) * 312, dtype=U64)
    x[:312] = state
    for b in range(312, len(x), 312):
        o = x[b - 312:b]
        x[b:b + 156] = twist(o[:156], o[1:157], o[156:312])
        x[b + 156:b + 311] = twist(o[156:311], o[157:312], x[b:b + 155])
        x[b + 311] = twist(o[311:312], x[b:b + 1], x[b + 155:b + 156])[0]
    return x[:312 + n]


def temper(x):
    x = x ^ ((x >> U64(29)) & U64(0x5555555555555555))
    x = x ^ ((x << U64(17)) & U64(0x71D67FFFEDA60000))
    x = x ^ ((x << U64(37)) & U64(0xFFF7EEE000000000))
    return x ^ (x >> U64(43))


def jump_poly(steps):
    out = (C.c_uint64 * 312)()
    assert pe.lib().sf_mt_jump_poly(C.c_uint64(steps), out) == 0
    words = np.frombuffer(out, dtype=U64)
    return np.nonzero(np.unpackbits(words.view(np.uint8), bitorder="little"))[0]


def test_numpy_generator_is_std_mt19937_64():
    # the C++ standard pins the 10000th output of a default-constructed engine
    x = raw(seed_state(5489), 10000)
    assert int(temper(x[312 + 9999:312 + 10000])[0]) == 9981545732273789042


@pytest.mark.parametrize("steps", [1, 1000, 624 * 37, 1 << 20])
def test_jumped_state_continues_the_stream(steps):
    t0 = time.time()
    terms = jump_poly(steps)
    assert time.time() - t0 < 30.0
    assert terms.max() < 19937
    s0 = seed_state(0x5DEECE66D)
    base = raw(s0, 19937 + 312)
    jumped = np.bitwise_xor.reduce(base[terms[:, None] + np.arange(312)[None, :]], axis=0)
    direct = raw(s0, steps + 2000)
    # the state is 19937 bits: x[W] contributes its upper 33 bits only
    assert np.array_equal(jumped[1:], direct[steps + 1:steps + 312])
    assert int((jumped[0] ^ direct[steps]) & UPPER) == 0
    cont = raw(jumped, 2000)
    assert np.array_equal(cont[312:], direct[steps + 312:steps + 2312])


def test_jump_poly_rejects_null():
    assert pe.lib().sf_mt_jump_poly(C.c_uint64(5), None) != 0
