# baseline-policy device parity + experiment tests, then the 888-instance econoserve probe (regression check)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_baselines.py tests/test_experiment.py tests/test_known_answers.py -m gpu -x -q > gpurun_out/bl_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bl_pytest.log
timeout 900 python tools/probe_scale.py --counts 888 --iters 1000 --lanes 0 > gpurun_out/bl_probe_scale.log 2>&1
