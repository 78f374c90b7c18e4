#!/usr/bin/env bash
# Collect the round's profiling evidence on a B200 (run under gpurun; single GPU).
#   1. launch list of the bench command (per-kernel device time, cold/serialised)
#   2. one `ncu --set full` capture of K1 (k_window_bounds, k_route_bin) and K2
#   3. one capture of the decode kernels (K3a k_tbt_p95 / k_tps, K3b k_decode_replay)
#   4. one capture of the closed-loop decode pool (K5 k_decode_pool)
# Outputs go to gpurun_out/; tools/summarize_profiles.py turns them into profiles/<round>_*.
# <round>_units.json records the work units of each captured launch (trajectories, scenarios)
# so bench.py can turn ncu instruction counts into per-unit issue-slot rooflines.
set -u
ROUND=${1:-r2}
DEC_SCEN=20000
POOL_SCEN=2000
mkdir -p gpurun_out
echo "{\"k_decode_replay\": $((DEC_SCEN * 4)), \"k_decode_pool\": ${POOL_SCEN}}" > gpurun_out/${ROUND}_units.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${ROUND}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/${ROUND}_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_route_bin|k_prefill_select|k_window_bounds|k_summary|k_cells_finish|k_prefill_pass" -s 12 -c 7 \
    -o gpurun_out/${ROUND}_prefill python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph \
    --scenarios 2000 --pool-scenarios 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_decode_replay|k_tbt_p95|k_tps" -s 3 -c 3 \
    -o gpurun_out/${ROUND}_decode python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph \
    --scenarios ${DEC_SCEN} --pool-scenarios 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_decode_pool" -s 2 -c 2 \
    -o gpurun_out/${ROUND}_pool python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph \
    --scenarios 2000 --pool-scenarios ${POOL_SCEN} > /dev/null 2>&1
ls -la gpurun_out/${ROUND}_*
