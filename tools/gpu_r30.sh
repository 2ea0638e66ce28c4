timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r30_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r30_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r30_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r30_smoke.log
cat > /tmp/cfg.json <<'J'
{"trace": {"synthetic": {"n_requests": 2000, "arrival_rate": 40.0}}, "policies": ["econoserve-full", "econoserve-sd", "econoserve-d"],
 "kvc": {"capacity": 14648, "block_size": 16}, "predictor": {"model": "bucket", "accuracy": 0.775, "tolerance": 0.1}, "sweep": {"reserved_fraction": [0.03, 0.06], "slo_scale": [1.0, 2.0]}}
J
(timeout 300 python -m paper_2411_06364_b200 run -c /tmp/cfg.json -o gpurun_out/r30_run && timeout 300 python -m paper_2411_06364_b200 sweep -c /tmp/cfg.json -o gpurun_out/r30_sweep.csv) > gpurun_out/r30_cli.log 2>&1; echo "cli rc=$?" >> gpurun_out/r30_cli.log
