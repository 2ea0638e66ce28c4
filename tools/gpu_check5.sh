mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/chk6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk6_pytest.log
for r in 1 2 3; do
  ECONO_VERBOSE=1 timeout 900 python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/chk6_bench_$r.json 2> gpurun_out/chk6_bench_$r.err
done
