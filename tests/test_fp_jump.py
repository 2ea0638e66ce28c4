"""The closed-form jump over repeated floating-point additions used by the
quiet-span replay (engine.cuh fp_repeat_add) equals k sequential adds bit for
bit: random magnitudes, exact ties, binade crossings, subnormals, zero."""
import ctypes as C
import os
import struct

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOSTSIM = os.path.join(ROOT, "tests", "_hostsim", "libeconoserve_hostsim.so")


def _lib():
    L = C.CDLL(HOSTSIM)
    L.econo_hostsim_repeat_add.argtypes = [C.c_double, C.c_double, C.c_int64]
    L.econo_hostsim_repeat_add.restype = C.c_double
    return L


def seq(x, d, k):
    for _ in range(k):
        x = x + d
    return x


def bits(v):
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def test_repeat_add_matches_sequential():
    L = _lib()
    rng = np.random.default_rng(5)
    cases = [(0.0, 0.0055, 1000), (0.0, 0.0, 10), (1.0, 1e-17, 100), (1.0, 2 ** -53, 9), (1.0, 3 * 2 ** -53, 9),
             (2.0 ** 52 - 3, 1.0, 10), (1.0, 0.5, 7), (5e-324, 5e-324, 50), (0.0, 5e-324, 3), (1.5, 2 ** -53, 8),
             (1.0, 2 ** -52 + 2 ** -53, 11), (7.0, 1.5, 40), (0.1, 0.1, 100), (123.456, 0.0051, 5000)]
    for _ in range(3000):
        x = float(rng.choice([0.0, rng.random(), rng.random() * 1e3, rng.random() * 1e-3, rng.random() * 1e6]))
        d = float(rng.choice([rng.random() * 1e-2, rng.random(), rng.random() * 1e-9, 0.005 + rng.random() * 1e-3]))
        cases.append((x, d, int(rng.integers(0, 3000))))
    for t in range(20000):  # clock / execution_time shapes: dt-like steps from 0 or small starts
        x = 0.0 if t % 5 == 0 else float(rng.random() * rng.choice([1e-3, 1.0, 10.0, 100.0, 1e5]))
        d = float(rng.choice([0.005 + rng.integers(1, 200) * 1e-4, rng.random(), rng.random() * 1e-6]))
        cases.append((x, d, int(rng.integers(1, 400))))
    for _ in range(2000):  # ties: d an odd multiple of half an ulp of x
        e = int(rng.integers(-20, 20))
        x = float(np.ldexp(1.0 + rng.integers(0, 2 ** 20) * 2.0 ** -20, e))
        u = float(np.ldexp(1.0, e - 52))
        d = u * (int(rng.integers(0, 64)) + 0.5)
        cases.append((x, d, int(rng.integers(1, 500))))
    bad = [(x, d, k) for x, d, k in cases if bits(L.econo_hostsim_repeat_add(x, d, k)) != bits(seq(x, d, k))]
    assert not bad, bad[:5]
