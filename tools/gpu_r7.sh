set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r7_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r7_pytest_gpu.log
timeout 900 python tools/probe_report.py > gpurun_out/r7_report.log 2>&1; echo "rc=$?" >> gpurun_out/r7_report.log
