"""Python host mirror of econosim::Engine over the C-ABI (include/econoserve_b200.h).

`Engine(trace, options)` / `step()` / `run()` / `report()` / `events()` /
`samples()` / `requests()`-style snapshots follow the reference's public
surface (engine.hpp:79-145); `run(trace, options)` is the one-call entry point
(engine.hpp:1039-1042). Errors raise `ConfigError` / `SimulationError` with the
reference's messages (common.hpp:17-24).

The library is the sm_100a build in paper_2411_06364_b200/_lib/. There is no CPU
fallback: without a CUDA device, creating an Engine raises DeviceError.
"""
import ctypes as C
import os

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libeconoserve_b200.so")
# development builds (e.g. the per-phase cycle counters, tools/gpu_phases.sh)
# are loaded by pointing ECONO_LIB at them; the default is the product build
if os.environ.get("ECONO_LIB"):
    LIB_PATH = os.environ["ECONO_LIB"]

SYMBOLS = [
    "econo_default_options", "econo_create", "econo_step", "econo_run", "econo_records",
    "econo_report", "econo_events", "econo_samples", "econo_scalars", "econo_snapshot",
    "econo_destroy", "econo_instance_bytes", "econo_batch_create", "econo_batch_create_soa", "econo_batch_launch", "econo_batch_launch_slice",
    "econo_batch_launch_to", "econo_batch_sync",
    "econo_batch_scalars", "econo_batch_engine", "econo_batch_partials", "econo_batch_destroy",
    "econo_generate_trace", "econo_batch_checkpoint", "econo_batch_restore", "econo_batch_debug",
    "econo_batch_reports", "econo_batch_jct_prepare", "econo_batch_jct_hist", "econo_batch_jct_percentiles",
    "econo_jct_key_to_double", "econo_batch_ingest", "econo_libm_eval",
]


class ConfigError(ValueError):
    """econosim::ConfigError (common.hpp:17-19)."""


class SimulationError(RuntimeError):
    """econosim::SimulationError (common.hpp:22-24)."""


class DeviceError(RuntimeError):
    """No usable CUDA device / CUDA failure (the product has no CPU path)."""


def _raise(rc, err):
    msg = err.value.decode(errors="replace")
    if rc == abi.ECONFIG:
        raise ConfigError(msg)
    if rc == abi.ESIM:
        raise SimulationError(msg)
    raise DeviceError(msg)


_libs = {}


def load(path=None):
    """Loads (once) and types the C-ABI library at `path` (default: the sm_100a build)."""
    path = path or LIB_PATH
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise DeviceError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(path)
    vp, i64, i32, cp, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_char_p, C.c_size_t
    L.econo_default_options.argtypes = [C.POINTER(abi.Options)]
    L.econo_create.argtypes = [vp, i64, C.POINTER(abi.Options), C.c_int, C.POINTER(vp), cp, sz]
    L.econo_step.argtypes = [vp, i64, C.POINTER(i32), cp, sz]
    L.econo_run.argtypes = [vp, cp, sz]
    L.econo_records.argtypes = [vp, vp, i64, cp, sz]
    L.econo_report.argtypes = [vp, C.POINTER(abi.Report), cp, sz]
    L.econo_events.argtypes = [vp, vp, i64]
    L.econo_events.restype = i64
    L.econo_samples.argtypes = [vp, vp, i64]
    L.econo_samples.restype = i64
    L.econo_scalars.argtypes = [vp, C.POINTER(abi.Scalars)]
    L.econo_snapshot.argtypes = [vp, vp, i64]
    L.econo_snapshot.restype = i64
    L.econo_destroy.argtypes = [vp]
    L.econo_instance_bytes.argtypes = [vp, i64, C.POINTER(abi.Options), C.c_char_p, C.c_size_t]
    L.econo_instance_bytes.restype = i64
    L.econo_batch_create.argtypes = [C.POINTER(vp), C.POINTER(i64), i32, C.POINTER(abi.Options),
                                     C.c_int, C.POINTER(vp), cp, sz]
    L.econo_batch_create_soa.argtypes = [C.POINTER(abi.TraceSoA), C.POINTER(i64), i32, C.POINTER(abi.Options),
                                         C.c_int, C.POINTER(vp), cp, sz]
    L.econo_batch_launch.argtypes = [vp, i64, vp]
    L.econo_batch_launch_slice.argtypes = [vp, i64, i64, vp]
    L.econo_batch_launch_to.argtypes = [vp, i64, i64, vp]
    L.econo_libm_eval.argtypes = [i32, vp, vp, i64, C.c_int, cp, sz]
    L.econo_batch_sync.argtypes = [vp, cp, sz]
    L.econo_batch_scalars.argtypes = [vp, C.POINTER(abi.Scalars)]
    L.econo_batch_engine.argtypes = [vp, i32, C.POINTER(vp)]
    L.econo_batch_partials.argtypes = [vp, vp, cp, sz]
    L.econo_batch_destroy.argtypes = [vp]
    L.econo_batch_checkpoint.argtypes = [vp, cp, sz]
    L.econo_batch_restore.argtypes = [vp, cp, sz]
    L.econo_batch_debug.argtypes = [vp, vp]
    L.econo_batch_reports.argtypes = [vp, vp, cp, sz]
    L.econo_batch_ingest.argtypes = [vp, cp, sz]
    L.econo_batch_jct_prepare.argtypes = [vp, cp, sz]
    L.econo_batch_jct_hist.argtypes = [vp, i32, vp, i32, i32, vp, cp, sz]
    L.econo_batch_jct_percentiles.argtypes = [vp, vp, i32, vp, cp, sz]
    L.econo_jct_key_to_double.argtypes = [C.c_uint64]
    L.econo_jct_key_to_double.restype = C.c_double
    L.econo_generate_trace.argtypes = [i64, C.c_double, C.POINTER(abi.LengthDist),
                                       C.POINTER(abi.LengthDist), C.c_uint64, vp, cp, sz]
    _libs[path] = L
    return L


def instance_bytes(trace, options, lib=None):
    """HBM bytes one instance of `trace` occupies (econo_instance_bytes)."""
    L = load(lib)
    t = abi.trace_array(trace)
    err = C.create_string_buffer(1024)
    o = options
    r = L.econo_instance_bytes(t.ctypes.data, len(t), C.byref(o), err, 1024)
    if r < 0:
        _raise(int(-r), err)
    return int(r)


def generate_trace(n, rate, prompt, rl, seed, lib=None, out=None):
    """generate_synthetic (workload.hpp:104-125): host-side input preparation.
    `out` (optional): a preallocated TRACE_DTYPE array of n records, e.g. a view
    of pinned host memory so the upload runs at full link speed."""
    L = load(lib)
    if out is None:
        out = np.zeros(n, dtype=abi.TRACE_DTYPE)
    elif out.dtype != abi.TRACE_DTYPE or len(out) != n or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous TRACE_DTYPE array of n records")
    err = C.create_string_buffer(512)
    rc = L.econo_generate_trace(n, rate, C.byref(abi.LengthDist(*prompt)),
                                C.byref(abi.LengthDist(*rl)), seed, out.ctypes.data, err, 512)
    if rc:
        _raise(rc, err)
    return out


class Engine:
    """econosim::Engine (engine.hpp:79-145) running on the B200."""

    def __init__(self, trace, options=None, device=0, lib=None):
        self._L = load(lib)
        self.trace = abi.trace_array(trace)
        self.options = options if options is not None else abi.default_options()
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = self._L.econo_create(self.trace.ctypes.data, len(self.trace), C.byref(self.options),
                                  device, C.byref(h), err, 1024)
        if rc:
            _raise(rc, err)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self._L.econo_destroy(self.h)
            self.h = None

    __del__ = close

    def step(self, n=1):
        """Advances up to n Engine::step() calls; returns step()'s last value."""
        more = C.c_int32()
        err = C.create_string_buffer(1024)
        rc = self._L.econo_step(self.h, n, C.byref(more), err, 1024)
        if rc:
            _raise(rc, err)
        return bool(more.value)

    def run(self):
        err = C.create_string_buffer(1024)
        rc = self._L.econo_run(self.h, err, 1024)
        if rc:
            _raise(rc, err)
        return self.report()

    def records(self):
        out = np.zeros(len(self.trace), dtype=abi.RECORD_DTYPE)
        err = C.create_string_buffer(1024)
        rc = self._L.econo_records(self.h, out.ctypes.data, len(out), err, 1024)
        if rc:
            _raise(rc, err)
        return out

    def report(self):
        """(records, EconoReport) — finalize() + aggregate() (engine.hpp:963-994)."""
        recs = self.records()
        rep = abi.Report()
        err = C.create_string_buffer(1024)
        rc = self._L.econo_report(self.h, C.byref(rep), err, 1024)
        if rc:
            _raise(rc, err)
        return recs, rep

    finalize = report

    def events(self):
        n = self._L.econo_events(self.h, None, 0)
        out = np.zeros(n, dtype=abi.EVENT_DTYPE)
        self._L.econo_events(self.h, out.ctypes.data, n)
        return out

    def samples(self):
        n = self._L.econo_samples(self.h, None, 0)
        out = np.zeros(n, dtype=abi.SAMPLE_DTYPE)
        self._L.econo_samples(self.h, out.ctypes.data, n)
        return out

    def scalars(self):
        s = abi.Scalars()
        self._L.econo_scalars(self.h, C.byref(s))
        return s

    def snapshot(self):
        n = self._L.econo_snapshot(self.h, None, 0)
        out = np.zeros(n, dtype=np.int64)
        self._L.econo_snapshot(self.h, out.ctypes.data, n)
        return out

    # engine.hpp:136-145 accessors
    def clock(self):
        return self.scalars().clock

    def hosted_slots_created(self):
        return self.scalars().hosted_slots_created

    def hosted_overruns(self):
        return self.scalars().hosted_overruns

    def calibrated_prefill_time(self):
        return self.scalars().calibrated_prefill_time

    def calibrated_decode_time(self):
        return self.scalars().calibrated_decode_time


def run(trace, options=None, device=0, lib=None):
    """econosim::run(trace, opt) (engine.hpp:1039-1042)."""
    return Engine(trace, options, device=device, lib=lib).run()


class Batch:
    """Many independent instances advanced together (one warp each) — the
    device form of run_sweep's engine pool (sweep.hpp:112-149)."""

    def __init__(self, traces, options, device=0, lib=None):
        """traces: records (TRACE_DTYPE arrays, econo_batch_create) or, all of
        them, abi.SoaTrace columns (econo_batch_create_soa: 16 B per request
        copied straight into the device layout)."""
        self._L = load(lib)
        soa = len(traces) > 0 and all(isinstance(t, abi.SoaTrace) for t in traces)
        self.traces = list(traces) if soa else [abi.trace_array(t) for t in traces]
        if not isinstance(options, (list, tuple)):
            options = [options] * len(self.traces)
        self.options = (abi.Options * len(self.traces))(*options)
        ns = (C.c_int64 * len(self.traces))(*[len(t) for t in self.traces])
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        if soa:
            arr = (abi.TraceSoA * len(self.traces))(*[t.struct() for t in self.traces])
            rc = self._L.econo_batch_create_soa(arr, ns, len(self.traces), self.options, device,
                                                C.byref(h), err, 1024)
        else:
            ptrs = (C.c_void_p * len(self.traces))(*[t.ctypes.data for t in self.traces])
            rc = self._L.econo_batch_create(ptrs, ns, len(self.traces), self.options, device,
                                            C.byref(h), err, 1024)
        if rc:
            _raise(rc, err)
        self.h = h
        self.n = len(self.traces)

    def close(self):
        if getattr(self, "h", None):
            self._L.econo_batch_destroy(self.h)
            self.h = None

    __del__ = close

    def launch(self, max_steps, stream=None, slice_ns=0):
        if slice_ns:
            self._L.econo_batch_launch_slice(self.h, max_steps, int(slice_ns), stream)
        else:
            self._L.econo_batch_launch(self.h, max_steps, stream)

    def launch_to(self, target_steps, stream=None, slice_ns=0):
        """Advance every instance until it has made target_steps step() calls
        in total (econo_batch_launch_to), time-sliced when slice_ns > 0."""
        rc = self._L.econo_batch_launch_to(self.h, int(target_steps), int(slice_ns), stream)
        if rc:
            raise ConfigError("econo_batch_launch_to: negative target")

    def advance_to(self, target_steps, stream=None, slice_ns=0):
        """launch_to repeated until every live instance reached the target
        (or finished / faulted); synchronises."""
        while True:
            self.launch_to(target_steps, stream, slice_ns)
            self.sync()
            if all(s.steps >= target_steps or s.done or s.error for s in self.scalars()):
                return

    def sync(self):
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_sync(self.h, err, 1024)
        if rc:
            _raise(rc, err)

    def scalars(self):
        out = (abi.Scalars * self.n)()
        self._L.econo_batch_scalars(self.h, out)
        return list(out)

    def checkpoint(self):
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_checkpoint(self.h, err, 1024)
        if rc:
            _raise(rc, err)

    def restore(self):
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_restore(self.h, err, 1024)
        if rc:
            _raise(rc, err)

    def debug(self):
        out = np.zeros((self.n, abi.DEBUG_WORDS), dtype=np.int64)
        self._L.econo_batch_debug(self.h, out.ctypes.data)
        return out

    def ingest(self):
        """Grid-wide ingest of every instance's due arrivals (econo_batch_ingest)."""
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_ingest(self.h, err, 1024)
        if rc:
            _raise(rc, err)

    def snapshot(self, i):
        """Canonical state snapshot of instance i (econo_snapshot on a batch view)."""
        v = C.c_void_p()
        self._L.econo_batch_engine(self.h, i, C.byref(v))
        n = self._L.econo_snapshot(v, None, 0)
        out = np.zeros(n, dtype=np.int64)
        self._L.econo_snapshot(v, out.ctypes.data, n)
        return out

    def engine(self, i):
        """Borrowed single-engine view of instance i (econo_batch_engine)."""
        v = C.c_void_p()
        self._L.econo_batch_engine(self.h, i, C.byref(v))
        return v

    def records(self, i):
        """finalize()'s per-request records of instance i (engine.hpp:963-994)."""
        out = np.zeros(len(self.traces[i]), dtype=abi.RECORD_DTYPE)
        err = C.create_string_buffer(1024)
        rc = self._L.econo_records(self.engine(i), out.ctypes.data, len(out), err, 1024)
        if rc:
            _raise(rc, err)
        return out

    def reports(self):
        """aggregate() per instance, on the device (econo_batch_reports)."""
        out = (abi.Report * self.n)()
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_reports(self.h, out, err, 1024)
        if rc:
            _raise(rc, err)
        return list(out)

    def jct_percentiles(self, qs):
        """Exact per-instance percentile() of JCT (metrics.hpp:81-89): (n_inst, len(qs))."""
        q = np.asarray(qs, dtype=np.float64)
        out = np.zeros((self.n, len(q)), dtype=np.float64)
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_jct_percentiles(self.h, q.ctypes.data, len(q), out.ctypes.data, err, 1024)
        if rc:
            _raise(rc, err)
        return out

    def jct_prepare(self):
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_jct_prepare(self.h, err, 1024)
        if rc:
            _raise(rc, err)

    def jct_hist(self, prefixes, consumed_bits, digit_bits):
        """One radix-select pass over all instances: (len(prefixes), 2**digit_bits) counts."""
        pf = np.ascontiguousarray(prefixes, dtype=np.uint64)
        out = np.zeros((len(pf), 1 << digit_bits), dtype=np.uint64)
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_jct_hist(self.h, len(pf), pf.ctypes.data, consumed_bits, digit_bits,
                                          out.ctypes.data, err, 1024)
        if rc:
            _raise(rc, err)
        return out

    def key_to_double(self, key):
        return self._L.econo_jct_key_to_double(int(key))

    def partials(self):
        out = np.zeros((self.n, abi.PARTIAL_WORDS), dtype=np.float64)
        err = C.create_string_buffer(1024)
        rc = self._L.econo_batch_partials(self.h, out.ctypes.data, err, 1024)
        if rc:
            _raise(rc, err)
        return out
