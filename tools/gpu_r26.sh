ECONO_PROF_PHASES=1 python -c "import __graft_entry__ as g; g.build_product()" > /dev/null 2>&1
timeout 900 python tools/probe_scale.py --counts 148 --iters 1000 --lanes 0 > gpurun_out/r26_scale_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/prof_cfg2 -f python tools/ncu_target.py --instances 64 --iters 1000 --n 100000 --workload cfg2_sharegpt_100k > gpurun_out/prof_cfg2.log 2>&1
