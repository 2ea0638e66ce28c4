mkdir -p gpurun_out
timeout 900 python tools/ab_multi.py --libs dt,rp --rounds 1 --slice-us 20000 --launches 3 > gpurun_out/ab_r2y_cfg3.log 2>&1
timeout 1500 python tools/ab_multi.py --libs dt,rp --rounds 1 --workload cfg2_sharegpt_100k --instances 2368 --n 100000 --slice-us 20000 --launches 3 --check-step 2000 > gpurun_out/ab_r2y_cfg2.log 2>&1
timeout 1500 python tools/ab_multi.py --libs dt,rp --rounds 1 --workload cfg4_mixed_1m --instances 1036 --slice-us 20000 --launches 3 --check-step 2002 > gpurun_out/ab_r2y_cfg4.log 2>&1
