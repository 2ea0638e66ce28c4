# quick A/B: nolog GPU parity + the 888-instance probe
timeout 900 python -m pytest tests/test_nolog_parity.py tests/test_gpu_bulk_ingest.py -m gpu -x -q > gpurun_out/probe_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/probe_pytest.log
timeout 900 python tools/probe_scale.py --counts ${COUNTS:-888} --iters 1000 --lanes 0 > gpurun_out/probe_scale.log 2>&1
