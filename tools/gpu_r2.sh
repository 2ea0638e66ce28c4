set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
ECONO_VERBOSE=1 timeout 1500 python tools/probe_scale.py > gpurun_out/r2_scale.log 2>&1; echo "rc=$?" >> gpurun_out/r2_scale.log
ECONO_VERBOSE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "rc=$?" >> gpurun_out/r2_bench.err
