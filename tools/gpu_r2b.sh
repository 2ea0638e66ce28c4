# round 2: scale parity tests, bench with the parity block, phase profile, full ncu capture at the bench config
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_bulk_ingest.py tests/test_gpu_slices.py -x -q -v > gpurun_out/r2b_scale.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_scale.log
timeout 900 python bench.py --no-other-workloads --no-policy-sweep --no-full-runs > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "rc=$?" >> gpurun_out/r2b_bench.err
ECONO_LIB=tools/_prof/libeconoserve_prof.so timeout 900 python tools/probe_scale.py --counts 1184 --iters 1000 > gpurun_out/r2b_phases.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/r2b_steps -f python tools/ncu_target.py --instances 1184 --slice-us 250 > gpurun_out/r2b_steps.log 2>&1
