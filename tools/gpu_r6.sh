set -x
timeout 900 python -m pytest tests/test_metrics_report.py tests/test_gpu_metrics.py -m gpu -x -q > gpurun_out/r6_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r6_pytest_gpu.log
timeout 900 python tools/probe_report.py > gpurun_out/r6_report.log 2>&1; echo "rc=$?" >> gpurun_out/r6_report.log
