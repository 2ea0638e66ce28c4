# A/B of two builds on the three BASELINE shapes (A, B: tools/_prof/lib_<X>.so)
mkdir -p gpurun_out
timeout 900 python tools/ab_multi.py --libs ${A},${B} --rounds 1 --slice-us 20000 --launches 3 > gpurun_out/ab_${TAG}_cfg3.log 2>&1
timeout 1500 python tools/ab_multi.py --libs ${A},${B} --rounds 1 --workload cfg2_sharegpt_100k --instances 2368 --n 100000 --slice-us 20000 --launches 3 --check-step 2000 > gpurun_out/ab_${TAG}_cfg2.log 2>&1
timeout 1500 python tools/ab_multi.py --libs ${A},${B} --rounds 1 --workload cfg4_mixed_1m --instances 1036 --slice-us 20000 --launches 3 --check-step 2002 > gpurun_out/ab_${TAG}_cfg4.log 2>&1
