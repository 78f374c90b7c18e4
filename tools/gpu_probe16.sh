# K1a' probe width A/B: bounds parity under the 16-wide build, then the e2e probe of each build
mkdir -p gpurun_out
GSB_LIB=$PWD/paper_2508_16449_b200/lib/ab/libgsb_p4.so timeout 600 python -m pytest tests/test_gpu_bounds.py -x -q > gpurun_out/p16_tests.log 2>&1; echo rc=$? >> gpurun_out/p16_tests.log
: > gpurun_out/p16.log
for r in 1 2; do for v in p4 p8; do
  echo "== $v $r" >> gpurun_out/p16.log
  GSB_LIB=$PWD/paper_2508_16449_b200/lib/ab/libgsb_$v.so timeout 300 python tools/e2e_probe.py 2>&1 | grep 'K1a pinned\|upload ||\|full e2e\|chunks= [23] ' >> gpurun_out/p16.log
done; done
