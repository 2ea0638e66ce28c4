"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/liboracle.so, the C
restatement (oracle/econo_oracle.c) of the reference's EconoServe step."""
import ctypes as C
import os

import numpy as np

from paper_2411_06364_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.orc_create.argtypes = [C.c_void_p, C.c_int64, C.POINTER(abi.Options),
                                 C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_step.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.c_char_p, C.c_size_t]
        L.orc_events.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_events.restype = C.c_int64
        L.orc_samples.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_samples.restype = C.c_int64
        L.orc_finalize.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(abi.Report),
                                   C.c_char_p, C.c_size_t]
        L.orc_scalars.argtypes = [C.c_void_p, C.POINTER(abi.Scalars)]
        L.orc_snapshot.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_snapshot.restype = C.c_int64
        L.orc_generate_trace.argtypes = [C.c_int64, C.c_double, C.POINTER(abi.LengthDist),
                                         C.POINTER(abi.LengthDist), C.c_uint64, C.c_void_p,
                                         C.c_char_p, C.c_size_t]
        L.orc_mt_draws.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.orc_shuffle_indices.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.orc_predict.argtypes = [C.POINTER(abi.Options), C.c_uint64, C.c_void_p, C.c_int64,
                                  C.c_void_p]
        L.orc_predict.restype = C.c_int64
        _lib = L
    return _lib


class EngineError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def generate_trace(n, rate, prompt, rl, seed):
    out = np.zeros(n, dtype=abi.TRACE_DTYPE)
    err = C.create_string_buffer(512)
    rc = lib().orc_generate_trace(n, rate, C.byref(abi.LengthDist(*prompt)),
                                  C.byref(abi.LengthDist(*rl)), seed, out.ctypes.data, err, 512)
    if rc:
        raise EngineError(rc, err.value.decode())
    return out


def mt_draws(seed, n):
    out = np.zeros(n, dtype=np.uint64)
    lib().orc_mt_draws(seed, n, out.ctypes.data)
    return out


def shuffle_indices(seed, n):
    out = np.zeros(n, dtype=np.int64)
    lib().orc_shuffle_indices(seed, n, out.ctypes.data)
    return out


def predict(opts, seed, true_rl):
    t = np.ascontiguousarray(true_rl, dtype=np.int64)
    out = np.zeros(len(t), dtype=np.int64)
    lib().orc_predict(C.byref(opts), seed, t.ctypes.data, len(t), out.ctypes.data)
    return out


class OracleEngine:
    """C restatement of econosim::Engine (engine.hpp:79-145), econoserve family."""

    def __init__(self, trace, opts):
        self.trace = abi.trace_array(trace)
        self.opts = opts
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib().orc_create(self.trace.ctypes.data, len(self.trace), C.byref(opts),
                              C.byref(h), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def step(self, n=1):
        more = C.c_int32()
        err = C.create_string_buffer(1024)
        rc = lib().orc_step(self.h, n, C.byref(more), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        return bool(more.value)

    def run(self):
        while self.step(1 << 30):
            pass
        return self.finalize()

    def events(self):
        n = lib().orc_events(self.h, None, 0)
        out = np.zeros(n, dtype=abi.EVENT_DTYPE)
        lib().orc_events(self.h, out.ctypes.data, n)
        return out

    def samples(self):
        n = lib().orc_samples(self.h, None, 0)
        out = np.zeros(n, dtype=abi.SAMPLE_DTYPE)
        lib().orc_samples(self.h, out.ctypes.data, n)
        return out

    def finalize(self):
        recs = np.zeros(len(self.trace), dtype=abi.RECORD_DTYPE)
        rep = abi.Report()
        err = C.create_string_buffer(1024)
        rc = lib().orc_finalize(self.h, recs.ctypes.data, len(recs), C.byref(rep), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        return recs, rep

    def scalars(self):
        s = abi.Scalars()
        lib().orc_scalars(self.h, C.byref(s))
        return s

    def snapshot(self):
        n = lib().orc_snapshot(self.h, None, 0)
        out = np.zeros(n, dtype=np.int64)
        lib().orc_snapshot(self.h, out.ctypes.data, n)
        return out
