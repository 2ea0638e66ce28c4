# full device test suite + a quick bench line (no secondary sections)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_pytest.log
timeout 1200 python bench.py --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err
