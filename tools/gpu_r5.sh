set -x
nproc > gpurun_out/r5_nproc.txt
timeout 600 python -m pytest tests/test_gpu_metrics.py tests/test_nolog_parity.py -m gpu -x -q > gpurun_out/r5_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r5_pytest_gpu.log
ECONO_VERBOSE=1 timeout 1200 python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err; echo "rc=$?" >> gpurun_out/r5_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/r5_ref.json 2> gpurun_out/r5_ref.err; echo "rc=$?" >> gpurun_out/r5_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r5_launches.csv \
  python bench.py --no-cpu-baseline > gpurun_out/r5_launches_bench.json 2> gpurun_out/r5_launches_bench.err
