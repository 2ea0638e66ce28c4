# full ncu capture of one time-sliced k_engine_steps launch at the bench's density (8 instances per SM)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine_steps -s 5 -c 1 \
  -o gpurun_out/r2c_steps -f python tools/ncu_target.py --instances 1184 --n 100000 --slice-us 250 > gpurun_out/r2c_steps.log 2>&1
free -g > gpurun_out/r2c_mem.txt; nproc >> gpurun_out/r2c_mem.txt; lscpu | grep -i "model name\|flags" | cut -c1-300 >> gpurun_out/r2c_mem.txt
