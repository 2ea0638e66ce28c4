timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r27_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r27_pytest_gpu.log
timeout 600 python tools/probe_full.py > gpurun_out/r27_full.log 2>&1
