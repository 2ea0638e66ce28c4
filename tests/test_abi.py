"""The C-ABI drop-in boundary: the product library loads, exports every
symbol include/econoserve_b200.h declares, and fails loudly without a GPU
(there is no CPU path in the product)."""
import ctypes as C
import os
import re

import pytest

from paper_2411_06364_b200 import abi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "econoserve_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(econo_[a-z_]+)\s*\(", src)))


def test_header_declares_the_engine_surface():
    names = declared()
    for n in ["econo_create", "econo_step", "econo_run", "econo_records", "econo_report",
              "econo_events", "econo_samples", "econo_snapshot", "econo_destroy",
              "econo_batch_create", "econo_batch_launch", "econo_batch_partials"]:
        assert n in names


def test_product_library_exports_every_declared_symbol():
    L = C.CDLL(engine.LIB_PATH)
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing
    assert set(engine.SYMBOLS) <= set(declared())


def c_layout(struct, fields):
    """sizeof/offsetof as the C compiler sees include/econoserve_b200.h."""
    import subprocess
    import tempfile
    body = "\n".join(f'printf("%zu ", offsetof({struct}, {f}));' for f in fields)
    src = (f'#include <stdio.h>\n#include <stddef.h>\n#include "econoserve_b200.h"\n'
           f'int main(void){{ printf("%zu ", sizeof({struct})); {body} return 0; }}')
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        return [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]


@pytest.mark.parametrize("cname,pyt", [("EconoTraceRecord", abi.TraceRecord), ("EconoOptions", abi.Options),
                                       ("EconoEvent", abi.Event), ("EconoSample", abi.Sample),
                                       ("EconoRecord", abi.Record), ("EconoReport", abi.Report),
                                       ("EconoScalars", abi.Scalars), ("EconoLengthDist", abi.LengthDist),
                                       ("EconoTraceSoA", abi.TraceSoA)])
def test_struct_layouts_match_header(cname, pyt):
    names = [f for f, _ in pyt._fields_]
    got = c_layout(cname, names)
    assert got[0] == C.sizeof(pyt), (cname, got[0], C.sizeof(pyt))
    assert got[1:] == [getattr(pyt, f).offset for f in names]


def test_default_options_match_reference_defaults():
    o = abi.Options()
    engine.load().econo_default_options(C.byref(o))
    ref = abi.default_options()
    assert bytes(o) == bytes(ref)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(engine.DeviceError, match="no CPU fallback"):
        engine.Engine([(0.1, 10, 10)], abi.default_options())


def test_generate_trace_matches_reference_generator():
    import numpy as np
    from oracle import port
    from paper_2411_06364_b200 import workloads as W
    for name in ("cfg1_alpaca_10k", "cfg3_bookcorpus_1m"):
        c = W.CONFIGS[name]
        a = engine.generate_trace(3000, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 9)
        b = port.generate_trace(3000, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 9)
        assert np.array_equal(a, b)


def test_numpy_views_match_structs():
    assert abi.TRACE_DTYPE.itemsize == C.sizeof(abi.TraceRecord)
    assert abi.EVENT_DTYPE.itemsize == C.sizeof(abi.Event)
    assert abi.SAMPLE_DTYPE.itemsize == C.sizeof(abi.Sample)
    assert abi.RECORD_DTYPE.itemsize == C.sizeof(abi.Record)
    for dt, st in [(abi.EVENT_DTYPE, abi.Event), (abi.SAMPLE_DTYPE, abi.Sample),
                   (abi.RECORD_DTYPE, abi.Record)]:
        for f, _ in st._fields_:
            assert dt.fields[f][1] == getattr(st, f).offset, f
