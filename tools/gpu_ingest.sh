# Burst-ingest check and profile (range scans vs tile sorts): the ingest parity
# tests, the ingest wall time at the bench scale for both paths, the ncu launch
# list (time + DRAM bytes) of the ingest kernels, one full ncu capture of
# k_ingest_ranges. Usage (through gpurun): TAG=r2i bash tools/gpu_ingest.sh
T=${TAG:-ing}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bulk_ingest.py tests/test_gpu_parity_scale.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
ECONO_VERBOSE=1 timeout 900 python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > gpurun_out/${T}_ranges_wall.log 2>&1
ECONO_INGEST_TILES=1 ECONO_VERBOSE=1 timeout 900 python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > gpurun_out/${T}_tiles_wall.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ingest --csv \
  --log-file gpurun_out/${T}_ingest_launches.csv python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > gpurun_out/${T}_ncu_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ranges -c 1 -f \
  -o gpurun_out/${T}_ranges_full python tools/ncu_target.py --instances 148 --warmup 0 --launches 0 > gpurun_out/${T}_ncu_full.log 2>&1
