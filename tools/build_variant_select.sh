# build libgsb.so with extra nvcc defines for gsb_select.cu into lib/ab/libgsb_NAME.so (timing
# probes only): bash tools/build_variant_select.sh NAME -DFLAG ...
set -e
name=$1; shift
L=paper_2508_16449_b200/lib
mkdir -p $L/ab /tmp/abobj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -Iinclude "$@" -c -o /tmp/abobj/gsb_select_$name.o paper_2508_16449_b200/csrc/gsb_select.cu
objs=$(ls $L/obj/*.o | grep -v gsb_select.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/ab/libgsb_$name.so /tmp/abobj/gsb_select_$name.o $objs
