# A/B of the range-scan ingest variants (ballot multisplit vs __match_any_sync):
# parity of the bulk-ingest tests under both, wall time at the bench scale, ncu
# launch list of each, one full capture of the default. TAG=... bash tools/gpu_ingest_ab.sh
T=${TAG:-iab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bulk_ingest.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
ECONO_INGEST_MATCH=1 timeout 900 python -m pytest tests/test_gpu_bulk_ingest.py -q -x -k ranges > gpurun_out/${T}_pytest_match.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_match.log
ECONO_VERBOSE=1 timeout 900 python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > gpurun_out/${T}_ballot_wall.log 2>&1
ECONO_INGEST_MATCH=1 ECONO_VERBOSE=1 timeout 900 python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > gpurun_out/${T}_match_wall.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ingest --csv \
  --log-file gpurun_out/${T}_ballot_launches.csv python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > /dev/null 2>&1
ECONO_INGEST_MATCH=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ingest --csv \
  --log-file gpurun_out/${T}_match_launches.csv python tools/ncu_target.py --instances 1331 --warmup 0 --launches 0 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ranges -c 1 -f \
  -o gpurun_out/${T}_ranges_full python tools/ncu_target.py --instances 148 --warmup 0 --launches 0 > gpurun_out/${T}_ncu_full.log 2>&1
