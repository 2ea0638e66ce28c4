mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_smoke.log
timeout 900 python bench.py --no-other-workloads --no-policy-sweep --no-full-runs > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "rc=$?" >> gpurun_out/r2a_bench.err
