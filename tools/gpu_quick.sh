# quick GPU iteration: parity tests, a bench line, and a focused ncu capture of K1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:+-k "$TESTS"} > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/q_bench.log 2>&1; echo rc=$? >> gpurun_out/q_bench.log
if [ -n "${NCU_K:-}" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -s ${NCU_S:-4} -c ${NCU_C:-2} \
  -o gpurun_out/q_k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph --scenarios 2000 --pool-scenarios 200 > gpurun_out/q_ncu.log 2>&1
fi
