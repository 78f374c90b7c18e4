# round-2 final evidence (one gpurun call): GPU tests, smoke, the default bench line (with the
# CPU baseline), the reference arm, the C5 / C2 lines, then the ncu captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo rc=$? >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo rc=$? >> gpurun_out/f_bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/f_bench_reference.log 2>&1; echo rc=$? >> gpurun_out/f_bench_reference.log
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/f_bench_c5.log 2>&1; echo rc=$? >> gpurun_out/f_bench_c5.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 > gpurun_out/f_bench_c2.log 2>&1; echo rc=$? >> gpurun_out/f_bench_c2.log
bash tools/profile_round.sh ${ROUND:-r2} > gpurun_out/prof.log 2>&1
cuobjdump -sass paper_2508_16449_b200/lib/obj/gsb_select.o > gpurun_out/${ROUND:-r2}_select.sass 2>/dev/null
