# which round-2 change slowed the Poisson shapes: A/B on configs[1] (2368 x 100k) with whole single-engine runs; DADD probe
mkdir -p gpurun_out
./tools/_prof/dadd_probe > gpurun_out/r2l_dadd.log 2>&1
timeout 1500 python tools/ab_multi.py --libs uni,pt,mo,fz,pk --rounds 1 --workload cfg2_sharegpt_100k --instances 2368 --n 100000 --slice-us 20000 --launches 3 --check-step 2000 --full-run cfg1_alpaca_10k > gpurun_out/ab_r2l.log 2>&1
timeout 900 python tools/ab_multi.py --libs fz,pk --rounds 1 --slice-us 20000 --launches 3 > gpurun_out/ab_r2l_cfg3.log 2>&1
