# one ncu --set full capture of kernels matching NCU_K (skip NCU_S, count NCU_C) + source page
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -s ${NCU_S:-1} -c ${NCU_C:-1} \
  -o gpurun_out/n_k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph --scenarios 2000 --pool-scenarios 64 ${BENCH_ARGS:-} > gpurun_out/n_ncu.log 2>&1
ncu -i gpurun_out/n_k.ncu-rep --page raw --csv > gpurun_out/n_k_raw.csv 2>/dev/null
ncu -i gpurun_out/n_k.ncu-rep --page source --csv --print-source sass > gpurun_out/n_k_sass.csv 2>/dev/null
ncu -i gpurun_out/n_k.ncu-rep --page details --csv > gpurun_out/n_k_details.csv 2>/dev/null
