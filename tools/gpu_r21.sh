timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/prof_steps_r21 -f python tools/ncu_target.py --instances 64 --iters 1000 > gpurun_out/prof_steps_r21.log 2>&1
