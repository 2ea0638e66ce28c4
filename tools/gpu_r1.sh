set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r1_nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 900 python bench.py --instances 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench64.json 2> gpurun_out/r1_bench64.err; echo "rc=$?" >> gpurun_out/r1_bench64.err
timeout 1500 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err; echo "rc=$?" >> gpurun_out/r1_bench.err
tail -3 gpurun_out/*.log gpurun_out/*.err; cat gpurun_out/*.json
