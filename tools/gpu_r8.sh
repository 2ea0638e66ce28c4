set -x
timeout 900 python -m pytest tests/test_metrics_report.py tests/test_facade_cpp.py -m gpu -x -q > gpurun_out/r8_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r8_pytest_gpu.log
timeout 600 python tools/probe_report.py > gpurun_out/r8_report.log 2>&1; echo "rc=$?" >> gpurun_out/r8_report.log
timeout 1200 python bench.py > gpurun_out/r8_bench.json 2> gpurun_out/r8_bench.err; echo "rc=$?" >> gpurun_out/r8_bench.err
