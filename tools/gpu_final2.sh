mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final2_smoke.log
timeout 1800 python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo "rc=$?" >> gpurun_out/final2_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/final2_ref.json 2> gpurun_out/final2_ref.err; echo "rc=$?" >> gpurun_out/final2_ref.err
