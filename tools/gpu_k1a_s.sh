# K1a' block size A/B from device memory (GSB_BOUNDS=search) against the sampled K1a, k_ab timings
mkdir -p gpurun_out
: > gpurun_out/k1as.log
for r in 1 2; do
  echo "== sampled $r" >> gpurun_out/k1as.log
  GSB_BOUNDS=sampled timeout 300 python tools/k_ab.py 2>&1 | grep 'K1a \|K1 ' >> gpurun_out/k1as.log
  for f in paper_2508_16449_b200/lib/ab/*.so; do
    echo "== $(basename $f) search $r" >> gpurun_out/k1as.log
    GSB_BOUNDS=search GSB_LIB=$PWD/$f timeout 300 python tools/k_ab.py 2>&1 | grep 'K1a \|K1 ' >> gpurun_out/k1as.log
  done
done
for f in paper_2508_16449_b200/lib/ab/*.so; do
  echo "== $(basename $f) e2e" >> gpurun_out/k1as.log
  GSB_LIB=$PWD/$f timeout 300 python tools/e2e_probe.py 2>&1 | grep 'K1a pinned\|upload ||\|full e2e\|chunks= 3' >> gpurun_out/k1as.log
done
