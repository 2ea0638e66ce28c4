timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/prof_cfg2b -f python tools/ncu_target.py --instances 64 --iters 1000 --n 100000 --workload cfg2_sharegpt_100k > gpurun_out/prof_cfg2b.log 2>&1
