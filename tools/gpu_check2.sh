mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_pytest.log
timeout 900 python tools/ab_multi.py --libs C,D --rounds 2 > gpurun_out/abm2.log 2>&1
timeout 1200 python bench.py --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err
