# K5 A/B: the pool rate of the default build and of each lib/ab/*.so (bench.py, pool leg)
mkdir -p gpurun_out
: > gpurun_out/k5ab.log
for f in default paper_2508_16449_b200/lib/ab/*.so default paper_2508_16449_b200/lib/ab/*.so; do
  echo "== $f" >> gpurun_out/k5ab.log
  if [ $f = default ]; then unset GSB_LIB; else export GSB_LIB=$PWD/$f; fi
  timeout 300 python bench.py --no-cpu-baseline --steps 8 --warmup 3 2>&1 | grep -o '"pool": {"value": [0-9.]*' >> gpurun_out/k5ab.log
done
