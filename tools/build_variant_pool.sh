# build libgsb.so with extra nvcc defines for gsb_pool.cu into lib/ab/libgsb_NAME.so (timing
# probes only): bash tools/build_variant_pool.sh NAME -DFLAG ...
set -e
name=$1; shift
L=paper_2508_16449_b200/lib
mkdir -p $L/ab /tmp/abobj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -Iinclude "$@" -c -o /tmp/abobj/gsb_pool_$name.o paper_2508_16449_b200/csrc/gsb_pool.cu
objs=$(ls $L/obj/*.o | grep -v gsb_pool.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/ab/libgsb_$name.so /tmp/abobj/gsb_pool_$name.o $objs
