set -x
timeout 900 python tools/probe_scale.py --counts 740 --iters 1000,10000 --lanes 0 > gpurun_out/r12_scale.log 2>&1; echo "rc=$?" >> gpurun_out/r12_scale.log
