set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r18_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r18_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r18_bench.json 2> gpurun_out/r18_bench.err; echo "rc=$?" >> gpurun_out/r18_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r18_launches.csv \
  python bench.py --no-cpu-baseline > gpurun_out/r18_launches_bench.json 2> gpurun_out/r18_launches_bench.err
