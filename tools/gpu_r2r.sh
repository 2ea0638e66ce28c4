# validation of the fast-kernel build: smoke, device tests, bench, launch list
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2r_pytest.log
timeout 1800 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo "rc=$?" >> gpurun_out/r2r_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r_launches.csv \
  python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/r2r_launches_bench.json 2> gpurun_out/r2r_launches_bench.err
