mkdir -p gpurun_out
timeout 900 python tools/ab_multi.py --libs fast,fo2 --rounds 1 --slice-us 20000 --launches 3 > gpurun_out/ab_r2s_cfg3.log 2>&1
timeout 1500 python tools/ab_multi.py --libs fast,fo2 --rounds 1 --workload cfg2_sharegpt_100k --instances 2368 --n 100000 --slice-us 20000 --launches 3 --check-step 2000 > gpurun_out/ab_r2s_cfg2.log 2>&1
