timeout 1500 python bench.py > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err; echo "rc=$?" >> gpurun_out/r20_bench.err
