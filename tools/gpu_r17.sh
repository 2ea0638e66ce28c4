set -x
timeout 900 python -m pytest tests/test_gpu_bulk_ingest.py tests/test_nolog_parity.py -m gpu -x -q > gpurun_out/r17_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r17_pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r17_ingest_launches.csv \
  python tools/probe_scale.py --counts 148 --iters 100 --lanes 0 > gpurun_out/r17_ingest.log 2>&1
timeout 900 python tools/probe_scale.py --counts 740 --iters 1000 --lanes 0 > gpurun_out/r17_scale.log 2>&1
