# round 2 validation of the current build: smoke, device tests, bench (+ reference arm), ncu launch list, full ncu capture
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
timeout 1800 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo "rc=$?" >> gpurun_out/r2p_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/r2p_ref.json 2> gpurun_out/r2p_ref.err; echo "rc=$?" >> gpurun_out/r2p_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2p_launches.csv \
  python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/r2p_launches_bench.json 2> gpurun_out/r2p_launches_bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/r2p_steps -f python tools/ncu_target.py --instances 1184 --n 100000 --slice-us 250 > gpurun_out/r2p_steps.log 2>&1
