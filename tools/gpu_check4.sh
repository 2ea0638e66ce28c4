mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bulk_ingest.py tests/test_metrics_report.py tests/test_known_answers.py -m gpu -x -q > gpurun_out/chk4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk4_pytest.log
for r in 1 2 3; do
  ECONO_VERBOSE=1 timeout 900 python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/chk4_bench_$r.json 2> gpurun_out/chk4_bench_$r.err
done
