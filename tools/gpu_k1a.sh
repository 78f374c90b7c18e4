mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py > gpurun_out/k1a_e2e_3.log 2>&1; echo rc=$? >> gpurun_out/k1a_e2e_3.log
