mkdir -p gpurun_out
for rc in 256 128 96 64 32; do
echo "RC=$rc" >> gpurun_out/k5p.log
GSB_POOL_RUN_CAP=$rc timeout 300 python bench.py --no-cpu-baseline --steps 8 --warmup 3 2>&1 | grep -o '"pool": {"value": [0-9.]*' >> gpurun_out/k5p.log
done
