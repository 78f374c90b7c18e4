# pipelined host-buffer pass: tests, e2e probe, bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pass.py tests/test_gpu_bounds.py tests/test_boundary.py -x -q > gpurun_out/hp_tests.log 2>&1; echo rc=$? >> gpurun_out/hp_tests.log
timeout 300 python tools/e2e_probe.py > gpurun_out/hp_e2e.log 2>&1; echo rc=$? >> gpurun_out/hp_e2e.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/hp_bench.log 2>&1; echo rc=$? >> gpurun_out/hp_bench.log
