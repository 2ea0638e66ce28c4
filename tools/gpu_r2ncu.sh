mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/r2ncu_steps -f python tools/ncu_target.py --instances 1331 --n 100000 --slice-us 250 > gpurun_out/r2ncu_steps.log 2>&1
