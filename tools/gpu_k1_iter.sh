# K1 iteration: route_bin / pass / config parity tests, then graph-timed entry points
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pass.py tests/test_gpu_configs.py -x -q > gpurun_out/k1_tests.log 2>&1; echo rc=$? >> gpurun_out/k1_tests.log
timeout 300 python tools/k_probe.py > gpurun_out/k1_probe.log 2>&1; echo rc=$? >> gpurun_out/k1_probe.log
