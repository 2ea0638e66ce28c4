"""The device's glibc 2.39 exp/log port (csrc/glibc_libm.cuh) against the
host's libm, bit for bit: these feed the lognormal predictor
(llround(true_rl * exp(N)), workload.hpp:233-235) and the polar method's
log(r2) (random.tcc:1811-1844), where a 1-ulp difference can flip an integer
prediction. The CPU check compiles the port's source for the host (>1e8
inputs); the GPU check evaluates it on the B200 (econo_libm_eval)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2411_06364_b200", "csrc")
BUILD = os.path.join(ROOT, "tests", "_hostsim")


def _build(src, out, shared=False):
    os.makedirs(BUILD, exist_ok=True)
    cmd = ["g++", "-x", "c++", "-O2", "-mfma", "-ffp-contract=off", "-I" + CSRC, "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", src), "-o", os.path.join(BUILD, out), "-lm"]
    if shared:
        cmd[1:1] = ["-shared", "-fPIC"]
    subprocess.run(cmd, check=True)
    return os.path.join(BUILD, out)


def test_port_matches_host_libm_bit_for_bit():
    exe = _build("libm_check.c", "libm_check")
    out = subprocess.run([exe, "12000000"], capture_output=True, text=True, timeout=600)
    checked, bad = map(int, out.stdout.split()[-2:])
    assert checked > 100_000_000
    assert bad == 0, out.stdout


def _inputs(n, seed=7):
    rng = np.random.default_rng(seed)
    a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    r2 = a * a + b * b
    r2 = r2[(r2 <= 1.0) & (r2 > 0.0)]
    noise = rng.standard_normal(n) * rng.choice([0.1, 0.2, 0.3, 0.6], n)
    wide = rng.uniform(-750, 720, n)
    rbits = rng.integers(0, 2**63, n, dtype=np.uint64).view(np.float64)
    return (np.concatenate([noise, wide, rbits, np.array([0.0, -0.0, 1.0, np.inf, -np.inf, 709.78, -745.1])]),
            np.concatenate([r2, 1 + rng.uniform(-0.1, 0.1, n), rng.uniform(0, 1, n), np.abs(rbits),
                            np.array([1.0, 5e-324, 1e-310, np.inf, 0.0])]))


@pytest.mark.gpu
def test_device_port_matches_host_libm():
    from paper_2411_06364_b200 import engine
    L = engine.load()
    ref = C.CDLL(_build("libm_apply.c", "libm_apply.so", shared=True))
    for fn, x in enumerate(_inputs(4_000_000)):
        x = np.ascontiguousarray(x)
        dev, want = np.empty_like(x), np.empty_like(x)
        err = C.create_string_buffer(512)
        rc = L.econo_libm_eval(fn, x.ctypes.data, dev.ctypes.data, len(x), 0, err, 512)
        assert rc == 0, err.value
        ref.libm_apply(fn, C.c_void_p(x.ctypes.data), C.c_void_p(want.ctypes.data), C.c_int64(len(x)))
        same = (dev.view(np.uint64) == want.view(np.uint64)) | (np.isnan(dev) & np.isnan(want))
        assert same.all(), (fn, x[~same][:5], dev[~same][:5], want[~same][:5])
