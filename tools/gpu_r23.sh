timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r23_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r23_pytest_gpu.log
timeout 900 python tools/probe_scale.py --counts 740 --iters 1000 --lanes 0 > gpurun_out/r23_scale.log 2>&1
