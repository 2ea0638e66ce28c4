nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/r31_mem.txt
ECONO_VERBOSE=1 timeout 1200 python bench.py --instances 888 --no-cpu-baseline --no-full-runs > gpurun_out/r31_bench888.json 2> gpurun_out/r31_bench888.err; echo "rc=$?" >> gpurun_out/r31_bench888.err
