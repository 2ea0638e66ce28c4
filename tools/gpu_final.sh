# round-end evidence: full bench line, reference arm, ncu launch list (DRAM bytes) of the bench,
# one `ncu --set full` capture of k_engine_steps and of the HBM-bound kernels, smoke()
set -x
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 1800 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "rc=$?" >> gpurun_out/final_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "rc=$?" >> gpurun_out/final_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads --no-policy-sweep > gpurun_out/final_launches_bench.json 2> gpurun_out/final_launches_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/final_steps -f python tools/ncu_target.py --instances 148 --iters 1000 > gpurun_out/final_steps.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_radix_scatter|k_bulk_keys|k_partials_slices|k_jct_hist|k_init_req" -c 6 \
  -o gpurun_out/final_hbm -f python tools/probe_report.py > gpurun_out/final_hbm.log 2>&1
