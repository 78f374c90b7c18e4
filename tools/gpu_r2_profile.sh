# round-2 evidence: launch list, ncu captures (prefill, decode, pool), K2 SASS excerpt
mkdir -p gpurun_out
bash tools/profile_round.sh r2 > gpurun_out/prof.log 2>&1
cuobjdump -sass paper_2508_16449_b200/lib/obj/gsb_select.o > gpurun_out/r2_select.sass 2>/dev/null
