"""Wire formats either side of the scheduling path,
through the C-ABI (wire.cpp): the trace CSV loader/writer of
workload.hpp:127-194, the FNV-1a trace hash of metrics.hpp:320-328 and the
to_json(report).dump(indent) schema of metrics.hpp:181-240."""
import ctypes as C

import numpy as np

from . import abi
from .engine import ConfigError, _raise, load

POLICY_NAMES = ["orca", "vllm", "sarathi", "multires", "sync-coupled", "econoserve-d", "econoserve-sd",
                "econoserve-sdo", "econoserve-full"]


def _types(L):
    if getattr(L, "_wire_typed", False):
        return L
    i64, vp, cp, sz = C.c_int64, C.c_void_p, C.c_char_p, C.c_size_t
    L.econo_parse_trace_csv.argtypes = [cp, i64, cp, vp, i64, C.POINTER(i64), cp, sz]
    L.econo_load_trace_csv.argtypes = [cp, vp, i64, C.POINTER(i64), cp, sz]
    L.econo_write_trace_csv.argtypes = [vp, i64, cp, i64, C.POINTER(i64)]
    L.econo_trace_hash.argtypes = [vp, i64]
    L.econo_trace_hash.restype = C.c_uint64
    L.econo_json_double.argtypes = [C.c_double, cp, i64, C.POINTER(i64)]
    L.econo_report_to_json.argtypes = [cp, C.POINTER(abi.Report), vp, i64, cp, C.c_int32, cp, i64,
                                       C.POINTER(i64)]
    L._wire_typed = True
    return L


def _lib(lib=None):
    return _types(load(lib))


def parse_trace_csv(text, name="<stream>", lib=None):
    """load_trace_csv(istream, name): raises ConfigError with the reference's message."""
    L = _lib(lib)
    b = text.encode() if isinstance(text, str) else bytes(text)
    n = C.c_int64()
    err = C.create_string_buffer(1024)
    rc = L.econo_parse_trace_csv(b, len(b), name.encode(), None, 0, C.byref(n), err, 1024)
    if rc:
        _raise(rc, err)
    out = np.zeros(n.value, dtype=abi.TRACE_DTYPE)
    L.econo_parse_trace_csv(b, len(b), name.encode(), out.ctypes.data, n.value, C.byref(n), err, 1024)
    return out


def load_trace_csv(path, lib=None):
    """load_trace_csv(path) (workload.hpp:189-194)."""
    L = _lib(lib)
    n = C.c_int64()
    err = C.create_string_buffer(1024)
    rc = L.econo_load_trace_csv(path.encode(), None, 0, C.byref(n), err, 1024)
    if rc:
        _raise(rc, err)
    out = np.zeros(n.value, dtype=abi.TRACE_DTYPE)
    rc = L.econo_load_trace_csv(path.encode(), out.ctypes.data, n.value, C.byref(n), err, 1024)
    if rc:
        _raise(rc, err)
    return out


def _out_str(call):
    n = C.c_int64()
    call(None, 0, C.byref(n))
    buf = C.create_string_buffer(n.value + 1)
    call(buf, n.value + 1, C.byref(n))
    return buf.raw[:n.value].decode()


def write_trace_csv(trace, lib=None):
    L = _lib(lib)
    t = abi.trace_array(trace)
    return _out_str(lambda o, c, n: L.econo_write_trace_csv(t.ctypes.data, len(t), o, c, n))


def trace_hash(trace, lib=None):
    t = abi.trace_array(trace)
    return int(_lib(lib).econo_trace_hash(t.ctypes.data, len(t)))


def json_double(v, lib=None):
    L = _lib(lib)
    return _out_str(lambda o, c, n: L.econo_json_double(float(v), o, c, n))


def report_json(report, records=None, policy="econoserve-full", indent=-1, lib=None, _L=None, config_json=None):
    """to_json(report, with_records = records is not None).dump(indent); config_json: the
    pre-serialised "config" echo (experiment.config_json)."""
    L = _types(_L) if _L is not None else _lib(lib)
    recs = None if records is None else np.ascontiguousarray(records, dtype=abi.RECORD_DTYPE)
    ptr = None if recs is None else recs.ctypes.data
    nrec = 0 if recs is None else len(recs)
    cfg = None if config_json is None else config_json.encode()
    return _out_str(lambda o, c, n: L.econo_report_to_json(policy.encode(), C.byref(report), ptr, nrec, cfg,
                                                          indent, o, c, n))


def engine_report_json(engine, with_records=True, indent=-1):
    """The finished engine's report as the reference CLI writes it
    (to_json(report).dump(indent), tools/econosim.cpp:38)."""
    recs, rep = engine.report()
    return report_json(rep, recs if with_records else None, POLICY_NAMES[engine.options.policy], indent,
                       _L=engine._L)


__all__ = ["ConfigError", "parse_trace_csv", "load_trace_csv", "write_trace_csv", "trace_hash", "json_double",
           "report_json", "engine_report_json"]
