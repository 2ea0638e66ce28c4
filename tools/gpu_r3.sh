set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_pytest_gpu.log
timeout 1500 python tools/probe_scale.py --counts 444,740 --iters 100,1000 --lanes 0,8,32 > gpurun_out/r3_scale.log 2>&1; echo "rc=$?" >> gpurun_out/r3_scale.log
