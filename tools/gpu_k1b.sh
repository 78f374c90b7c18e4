# K1b iteration: parity of the default build, then an A/B of the lib/ab variants (k_ab, 2 rounds)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pass.py tests/test_gpu_configs.py tests/test_gpu_bounds.py -x -q > gpurun_out/k1b_tests.log 2>&1; echo rc=$? >> gpurun_out/k1b_tests.log
bash tools/gpu_ab.sh
