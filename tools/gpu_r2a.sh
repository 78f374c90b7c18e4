mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_tests.log 2>&1; echo rc=$? >> gpurun_out/t_tests.log
timeout 600 python bench.py > gpurun_out/t_bench.log 2>&1; echo rc=$? >> gpurun_out/t_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/t_ref.log 2>&1; echo rc=$? >> gpurun_out/t_ref.log
