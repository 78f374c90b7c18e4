# K5 A/B over (build, first-launch run cap): the pool rate from bench.py's pool leg, two rounds
mkdir -p gpurun_out
: > gpurun_out/k5ab2.log
for r in 1 2; do
for combo in default:32 minb6:32 minb6:16 minb6:24 minb4:32; do
  lib=${combo%%:*}; cap=${combo##*:}
  if [ $lib = default ]; then unset GSB_LIB; else export GSB_LIB=$PWD/paper_2508_16449_b200/lib/ab/libgsb_$lib.so; fi
  echo "== $lib cap=$cap round $r" >> gpurun_out/k5ab2.log
  GSB_POOL_RUN_CAP=$cap timeout 300 python bench.py --no-cpu-baseline --steps 4 --warmup 3 --scenarios 2000 2>&1 | grep -o '"pool": {"value": [0-9.]*' >> gpurun_out/k5ab2.log
done
done
