ECONO_VERBOSE=1 timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r19_bench.json 2> gpurun_out/r19_bench.err
