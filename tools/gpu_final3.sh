mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slices.py tests/test_nolog_parity.py -m gpu -x -q > gpurun_out/final3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final3_pytest.log
timeout 1800 python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; echo "rc=$?" >> gpurun_out/final3_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final3_launches.csv \
  python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/final3_launches_bench.json 2> gpurun_out/final3_launches_bench.err
