"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_ref/libecono_ref.so,
the unmodified reference simulator compiled by oracle/Makefile."""
import ctypes as C
import os

import numpy as np

from paper_2411_06364_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libecono_ref.so")
_lib = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_create.argtypes = [C.c_void_p, C.c_int64, C.POINTER(abi.Options),
                                 C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_clone.argtypes = [C.c_void_p]
        L.ref_clone.restype = C.c_void_p
        L.ref_step.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.c_char_p, C.c_size_t]
        L.ref_events.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_events.restype = C.c_int64
        L.ref_event_detail.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_size_t]
        L.ref_samples.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_samples.restype = C.c_int64
        L.ref_finalize.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(abi.Report),
                                   C.c_char_p, C.c_size_t]
        L.ref_report_json.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.c_int, C.c_int]
        L.ref_report_json.restype = C.c_int64
        L.ref_scalars.argtypes = [C.c_void_p, C.POINTER(abi.Scalars)]
        L.ref_snapshot.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_snapshot.restype = C.c_int64
        L.ref_generate_trace.argtypes = [C.c_int64, C.c_double, C.POINTER(abi.LengthDist),
                                         C.POINTER(abi.LengthDist), C.c_uint64, C.c_void_p,
                                         C.c_char_p, C.c_size_t]
        L.ref_trace_hash.argtypes = [C.c_void_p, C.c_int64]
        L.ref_trace_hash.restype = C.c_uint64
        L.ref_fast_ingest.argtypes = [C.c_void_p]
        L.ref_fast_ingest.restype = C.c_int64
        L.ref_idle_to_first_arrival.argtypes = [C.c_void_p]
        L.ref_time_steps.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_time_steps.restype = C.c_double
        L.ref_time_steps_parallel.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_int64,
                                              C.c_void_p]
        L.ref_time_steps_parallel.restype = C.c_double
        L.ref_mt_draws.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.ref_shuffle_indices.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.ref_predict.argtypes = [C.POINTER(abi.Options), C.c_uint64, C.c_void_p, C.c_int64,
                                  C.c_void_p]
        L.ref_predict.restype = C.c_int64
        L.ref_json_double.argtypes = [C.c_double, C.c_char_p, C.c_int64]
        L.ref_json_double.restype = C.c_int64
        L.ref_parse_csv.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_void_p, C.c_int64,
                                    C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]
        L.ref_write_csv.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_int64]
        L.ref_write_csv.restype = C.c_int64
        _lib = L
    return _lib


def mt_draws(seed, n):
    out = np.zeros(n, dtype=np.uint64)
    lib().ref_mt_draws(seed, n, out.ctypes.data)
    return out


def shuffle_indices(seed, n):
    out = np.zeros(n, dtype=np.int64)
    lib().ref_shuffle_indices(seed, n, out.ctypes.data)
    return out


def predict(opts, seed, true_rl):
    t = np.ascontiguousarray(true_rl, dtype=np.int64)
    out = np.zeros(len(t), dtype=np.int64)
    lib().ref_predict(C.byref(opts), seed, t.ctypes.data, len(t), out.ctypes.data)
    return out


class EngineError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def generate_trace(n, rate, prompt, rl, seed):
    out = np.zeros(n, dtype=abi.TRACE_DTYPE)
    err = C.create_string_buffer(512)
    rc = lib().ref_generate_trace(n, rate, C.byref(abi.LengthDist(*prompt)),
                                  C.byref(abi.LengthDist(*rl)), seed, out.ctypes.data, err, 512)
    if rc:
        raise EngineError(rc, err.value.decode())
    return out


def trace_hash(trace):
    t = abi.trace_array(trace)
    return int(lib().ref_trace_hash(t.ctypes.data, len(t)))


class RefEngine:
    """econosim::Engine (engine.hpp:79-145), the reference itself."""

    def __init__(self, trace, opts, _handle=None):
        self.trace = abi.trace_array(trace)
        self.opts = opts
        if _handle is not None:
            self.h = C.c_void_p(_handle)
            return
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib().ref_create(self.trace.ctypes.data, len(self.trace), C.byref(opts),
                              C.byref(h), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_destroy(self.h)
            self.h = None

    def clone(self):
        return RefEngine(self.trace, self.opts, _handle=lib().ref_clone(self.h))

    def step(self, n=1):
        more = C.c_int32()
        err = C.create_string_buffer(1024)
        rc = lib().ref_step(self.h, n, C.byref(more), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        return bool(more.value)

    def run(self):
        while self.step(1 << 30):
            pass
        return self.report()

    def events(self):
        n = lib().ref_events(self.h, None, 0)
        out = np.zeros(n, dtype=abi.EVENT_DTYPE)
        lib().ref_events(self.h, out.ctypes.data, n)
        return out

    def event_detail(self, i):
        buf = C.create_string_buffer(256)
        lib().ref_event_detail(self.h, i, buf, 256)
        k, d = buf.value.decode().split("|", 1)
        return k, d

    def samples(self):
        n = lib().ref_samples(self.h, None, 0)
        out = np.zeros(n, dtype=abi.SAMPLE_DTYPE)
        lib().ref_samples(self.h, out.ctypes.data, n)
        return out

    def finalize(self):
        recs = np.zeros(len(self.trace), dtype=abi.RECORD_DTYPE)
        rep = abi.Report()
        err = C.create_string_buffer(1024)
        rc = lib().ref_finalize(self.h, recs.ctypes.data, len(recs), C.byref(rep), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        return recs, rep

    def report(self):
        return self.finalize()

    def report_json(self, with_records=True, indent=-1):
        n = lib().ref_report_json(self.h, None, 0, int(with_records), indent)
        buf = C.create_string_buffer(n + 1)
        lib().ref_report_json(self.h, buf, n + 1, int(with_records), indent)
        return buf.value.decode()

    def scalars(self):
        s = abi.Scalars()
        lib().ref_scalars(self.h, C.byref(s))
        return s

    def snapshot(self):
        n = lib().ref_snapshot(self.h, None, 0)
        out = np.zeros(n, dtype=np.int64)
        lib().ref_snapshot(self.h, out.ctypes.data, n)
        return out

    def fast_ingest(self):
        return lib().ref_fast_ingest(self.h)

    def idle_to_first_arrival(self):
        return lib().ref_idle_to_first_arrival(self.h)

    def time_steps(self, steps):
        pt = C.c_int64()
        secs = lib().ref_time_steps(self.h, steps, C.byref(pt))
        return secs, pt.value


def json_double(v):
    """nlohmann::ordered_json(v).dump() (the reports' double printer)."""
    buf = C.create_string_buffer(64)
    n = lib().ref_json_double(float(v), buf, 64)
    return buf.value[:n].decode()


def parse_csv(text, name="<stream>"):
    """load_trace_csv on text: (trace, None) or (None, (code, message))."""
    b = text.encode() if isinstance(text, str) else text
    n = C.c_int64()
    err = C.create_string_buffer(1024)
    rc = lib().ref_parse_csv(b, len(b), name.encode(), None, 0, C.byref(n), err, 1024)
    if rc:
        return None, (rc, err.value.decode())
    out = np.zeros(n.value, dtype=abi.TRACE_DTYPE)
    lib().ref_parse_csv(b, len(b), name.encode(), out.ctypes.data, n.value, C.byref(n), err, 1024)
    return out, None


def write_csv(trace):
    t = abi.trace_array(trace)
    n = lib().ref_write_csv(t.ctypes.data, len(t), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib().ref_write_csv(t.ctypes.data, len(t), buf, n + 1)
    return buf.value[:n].decode()


def _str_call(fn, *args):
    n = fn(*args, None, 0)
    if n < 0:
        return None
    buf = C.create_string_buffer(n + 1)
    fn(*args, buf, n + 1)
    return buf.value[:n].decode()


def _exp_types():
    L = lib()
    if not getattr(L, "_exp_typed", False):
        L.ref_parse_config.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_experiment_report.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_int64]
        L.ref_experiment_report.restype = C.c_int64
        L.ref_render_table.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_render_table.restype = C.c_int64
        L.ref_sweep_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_sweep_csv.restype = C.c_int64
        L._exp_typed = True
    return L


def parse_config_error(config_text):
    """parse_config: None, or (code, message)."""
    err = C.create_string_buffer(1024)
    rc = _exp_types().ref_parse_config(config_text.encode(), err, 1024)
    return None if rc == 0 else (rc, err.value.decode())


def experiment_report(config_text, policy, with_records=True, indent=2):
    """to_json(run_experiment(parse_config(text))[policy]).dump(indent)."""
    return _str_call(_exp_types().ref_experiment_report, config_text.encode(), policy.encode(), int(with_records),
                     indent)


def render_table(config_text, baseline):
    return _str_call(_exp_types().ref_render_table, config_text.encode(), baseline.encode())


def sweep_csv(config_text):
    return _str_call(_exp_types().ref_sweep_csv, config_text.encode())
