# A/B of builds of libgsb.so in paper_2508_16449_b200/lib/ab/ (tools/build_variant.sh) on one
# box: tools/k_ab.py under each, two rounds
mkdir -p gpurun_out
: > gpurun_out/ab.log
for r in 1 2; do
  for f in paper_2508_16449_b200/lib/ab/*.so; do
    echo "== $(basename $f) $r" >> gpurun_out/ab.log
    GSB_LIB=$PWD/$f timeout 300 python tools/k_ab.py >> gpurun_out/ab.log 2>&1
  done
done
