# A/B of two builds of the product library on the same box (dev tool):
# _lib/libeconoserve_b200_A.so vs _lib/libeconoserve_b200_B.so, alternating.
for v in A B A B; do
  cp paper_2411_06364_b200/_lib/libeconoserve_b200_$v.so paper_2411_06364_b200/_lib/libeconoserve_b200.so
  echo "== $v" >> gpurun_out/ab.log
  timeout 600 python tools/probe_scale.py --counts ${COUNTS:-888} --iters 1000 --lanes 0 2>&1 | grep "inst=" >> gpurun_out/ab.log
done
