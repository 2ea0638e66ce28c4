"""Wire formats against the compiled reference
(oracle/_ref): nlohmann's double printer, to_json(report).dump(indent) byte
for byte, load_trace_csv's parse results and error messages, write_trace_csv
bytes and the FNV-1a trace hash."""
import struct

import numpy as np
import pytest

from conftest import HOSTSIM
from oracle import port, ref
from paper_2411_06364_b200 import abi, wire, workloads as W
from paper_2411_06364_b200.engine import ConfigError, Engine

from cases import catalogue

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _doubles(n, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2 ** 63 - 1, size=n, dtype=np.int64).astype(np.uint64)
    bits[::2] |= np.uint64(1) << np.uint64(63)
    out = list(bits.view(np.float64))
    out += list(rng.random(n) * 1000.0) + list(rng.random(n)) + list(rng.random(n) * 1e-6)
    out += list(np.round(rng.random(n) * 1e5) / (1 + rng.integers(0, 1000, n)))
    out += [0.0, -0.0, 1.0, -1.0, 0.1, 1e15, 1e16, 1e17, 1e-4, 1e-5, 123456789012345.0, 1234567890123456.0,
            5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 2.0 ** -1074, 2.0 ** 52, 2.0 ** 53 + 2,
            float("inf"), float("-inf"), float("nan"), 0.30000000000000004, 100.0, 1e21, 1e22, 9.5367431640625e-07]
    out += [struct.unpack("<d", struct.pack("<Q", (e << 52)))[0] for e in range(1, 2047)]  # powers of two
    return out


def test_json_double_matches_nlohmann():
    bad = []
    for v in _doubles(40000, 7):
        a, b = wire.json_double(v), ref.json_double(v)
        if a != b:
            bad.append((v, a, b))
    assert not bad, bad[:5]


CASES = catalogue(port.generate_trace)


@pytest.mark.parametrize("name,trace,opts", CASES[::3], ids=[c[0] for c in CASES[::3]])
def test_report_json_bytes(name, trace, opts):
    e = Engine(trace, opts, lib=HOSTSIM)
    e.run()
    r = ref.RefEngine(trace, opts)
    r.run()
    for rec in (True, False):
        for ind in (-1, 2):
            assert wire.engine_report_json(e, with_records=rec, indent=ind) == r.report_json(rec, ind), (rec, ind)


CSV_CASES = [
    "arrival_time,prompt_len,response_len\n0,5,7\n0.5,3,4\n",
    "arrival_time,prompt_len,response_len\r\n0,5,7\r\n\r\n1e-3,3,4\r\n",
    "arrival_time,prompt_len,response_len",
    "",
    "arrival,prompt_len,response_len\n0,1,1\n",
    "arrival_time,prompt_len,response_len\n0,5\n",
    "arrival_time,prompt_len,response_len\n0,5,7,\n",
    "arrival_time,prompt_len,response_len\nx,5,7\n",
    "arrival_time,prompt_len,response_len\n0,0,7\n",
    "arrival_time,prompt_len,response_len\n0,5,0\n",
    "arrival_time,prompt_len,response_len\n-1,5,7\n",
    "arrival_time,prompt_len,response_len\n1,5,7\n0.5,5,7\n",
    "arrival_time,prompt_len,response_len\n 0.25, 5, 7\n",
    "arrival_time,prompt_len,response_len\n0x10,+5,7\n",
    "arrival_time,prompt_len,response_len\n1e400,5,7\n",
    "arrival_time,prompt_len,response_len\n1e-320,5,7\n",
    "arrival_time,prompt_len,response_len\nnan,5,7\n1,2,3\n",
    "arrival_time,prompt_len,response_len\ninf,5,7\n",
    "arrival_time,prompt_len,response_len\n0,99999999999999999999,7\n",
    "arrival_time,prompt_len,response_len\n0,5 ,7\n",
    "arrival_time,prompt_len,response_len\n\n\n0,5,7",
]


@pytest.mark.parametrize("k", range(len(CSV_CASES)))
def test_parse_trace_csv_matches_reference(k):
    text = CSV_CASES[k]
    want, werr = ref.parse_csv(text, "t.csv")
    try:
        got, gerr = wire.parse_trace_csv(text, "t.csv"), None
    except ConfigError as ex:
        got, gerr = None, (2, str(ex))
    assert gerr == werr
    if want is not None:
        assert len(got) == len(want)
        assert got.tobytes() == want.tobytes()


def test_write_csv_and_hash_match_reference(tmp_path):
    c = W.CONFIGS["cfg2_sharegpt_100k"]
    t = port.generate_trace(3000, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 11)
    text = wire.write_trace_csv(t)
    assert text == ref.write_csv(t)
    assert wire.trace_hash(t) == ref.trace_hash(t)
    p = tmp_path / "trace.csv"
    p.write_text(text)
    back = wire.load_trace_csv(str(p))
    assert back.tobytes() == abi.trace_array(t).tobytes()  # %.17g round-trips
    with pytest.raises(ConfigError, match="cannot open trace file"):
        wire.load_trace_csv(str(tmp_path / "missing.csv"))
