timeout 600 python tools/probe_full.py > gpurun_out/r28_full_new.log 2>&1
cp paper_2411_06364_b200/_lib/libeconoserve_b200_old.so paper_2411_06364_b200/_lib/libeconoserve_b200.so
timeout 600 python tools/probe_full.py > gpurun_out/r28_full_old.log 2>&1
