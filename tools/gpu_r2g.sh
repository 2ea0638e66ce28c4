# A/B of the outlined-cold-path build (+ tile-local ingest) against the uniform build; rest of the device tests; phases
mkdir -p gpurun_out
timeout 1500 python tools/ab_multi.py --libs uni,cold --rounds 2 --slice-us 20000 --launches 3 > gpurun_out/ab_r2g.log 2>&1
ECONO_LIB=tools/_prof/libeconoserve_prof.so timeout 900 python tools/probe_scale.py --counts 1184 --iters 1000 > gpurun_out/r2g_phases.log 2>&1
ECONO_LIB=tools/_prof/lib_cold.so ECONO_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_bulk_ingest.py tests/test_libm_port.py tests/test_metrics_report.py tests/test_nolog_parity.py tests/test_oracle_golden.py tests/test_policy_fuzz.py tests/test_wire.py -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log
