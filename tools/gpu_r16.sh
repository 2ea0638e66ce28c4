set -x
INST=148 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r16_ingest_launches.csv \
  python tools/probe_scale.py --counts 148 --iters 100 --lanes 0 > gpurun_out/r16_ingest.log 2>&1
