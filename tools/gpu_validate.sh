# round-end validation: smoke(), the full device test suite, the bench line and the reference arm
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final4_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final4_pytest.log
timeout 1800 python bench.py > gpurun_out/final4_bench.json 2> gpurun_out/final4_bench.err; echo "rc=$?" >> gpurun_out/final4_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/final4_ref.json 2> gpurun_out/final4_ref.err; echo "rc=$?" >> gpurun_out/final4_ref.err
