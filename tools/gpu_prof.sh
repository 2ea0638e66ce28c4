# ncu evidence for the current build (run under gpurun)
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --no-cpu-baseline > gpurun_out/launches_bench.json 2> gpurun_out/launches_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine_steps -s 4 -c 1 \
  -o gpurun_out/prof_steps -f python tools/ncu_target.py --instances ${NCU_INST:-32} > gpurun_out/prof_steps.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_init -c 4 \
  -o gpurun_out/prof_init -f python tools/ncu_target.py --instances ${NCU_INST:-32} --warmup 0 --launches 0 > gpurun_out/prof_init.log 2>&1
ls -la gpurun_out
