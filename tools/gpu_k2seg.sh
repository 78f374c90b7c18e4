# K2 segmented scan: parity of the default build, then an A/B of the lib/ab variants
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pass.py tests/test_gpu_configs.py tests/test_gpu_entrypoints.py -x -q > gpurun_out/k2seg_tests.log 2>&1; echo rc=$? >> gpurun_out/k2seg_tests.log
bash tools/gpu_ab.sh
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/k2seg_bench.log 2>&1; echo rc=$? >> gpurun_out/k2seg_bench.log
