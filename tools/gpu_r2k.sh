# device tests on the fused-completion build (product lib rebuilt in place), then the bench
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k_pytest.log
timeout 1800 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "rc=$?" >> gpurun_out/r2k_bench.err
