set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r10_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r10_pytest_gpu.log
timeout 900 python tools/probe_scale.py --counts 740 --iters 1000 --lanes 0 > gpurun_out/r10_scale.log 2>&1; echo "rc=$?" >> gpurun_out/r10_scale.log
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_engine_steps -s 4 -c 1 \
  -o gpurun_out/prof_steps_r10 -f python tools/ncu_target.py --instances 64 --iters 1000 > gpurun_out/prof_steps_r10.log 2>&1
