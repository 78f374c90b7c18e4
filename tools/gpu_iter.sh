# iteration run: selected gpu tests, a bench line without CPU baseline, optional ncu of NCU_K
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:+-k "$TESTS"} > gpurun_out/i_tests.log 2>&1; echo rc=$? >> gpurun_out/i_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/i_bench.log 2>&1; echo rc=$? >> gpurun_out/i_bench.log
if [ -n "${NCU_K:-}" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -s ${NCU_S:-4} -c ${NCU_C:-2} \
  -o gpurun_out/i_k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph --scenarios 2000 --pool-scenarios 64 > gpurun_out/i_ncu.log 2>&1
ncu -i gpurun_out/i_k.ncu-rep --page raw --csv > gpurun_out/i_k_raw.csv 2>/dev/null
fi
if [ -n "${NCU_LAUNCH:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graph --scenarios 2000 --pool-scenarios 64 > /dev/null 2>&1
fi
