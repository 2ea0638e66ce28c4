# round-end validation of the product build: smoke(), the device test suite, the bench line,
# the reference arm, and the ncu launch list (per-launch time + DRAM bytes) of the bench.
# Usage (from the repo root, through gpurun): TAG=r2z bash tools/gpu_validate.sh
T=${TAG:-val}
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 1800 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "rc=$?" >> gpurun_out/${T}_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu-baseline --no-full-runs --no-other-workloads \
  --no-policy-sweep > gpurun_out/${T}_launches_bench.json 2> gpurun_out/${T}_launches_bench.err
