mkdir -p gpurun_out
timeout 900 python tools/ab_multi.py --libs nr2,fast --rounds 1 --slice-us 20000 --launches 3 > gpurun_out/ab_r2q_cfg3.log 2>&1
timeout 1500 python tools/ab_multi.py --libs nr2,fast --rounds 1 --workload cfg2_sharegpt_100k --instances 2368 --n 100000 --slice-us 20000 --launches 3 --check-step 2000 > gpurun_out/ab_r2q_cfg2.log 2>&1
timeout 1500 python tools/ab_multi.py --libs nr2,fast --rounds 1 --workload cfg4_mixed_1m --instances 1036 --slice-us 20000 --launches 3 --check-step 2002 > gpurun_out/ab_r2q_cfg4.log 2>&1
ECONO_LIB=tools/_prof/libeconoserve_prof.so timeout 900 python tools/probe_scale.py --counts 1184 --iters 1000 > gpurun_out/r2q_phases.log 2>&1
