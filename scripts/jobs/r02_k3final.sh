timeout 1200 python -m pytest tests/test_gpu_rowstats.py tests/test_gpu_sample.py tests/test_gpu_model_parity.py tests/test_gpu_model.py -x -q -m gpu > gpurun_out/k3f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k3f_tests.log
for n in 107 10 256; do timeout 300 python scripts/k3_probe.py $n 4 >> gpurun_out/k3f_probe.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stats -c 1 -o gpurun_out/r02_ncu_k3_final_535 python scripts/k3_probe.py 107 4 > gpurun_out/k3f_ncu.log 2>&1
WS_PROFILE_MODEL=1 timeout 300 python scripts/forward_probe.py 5 > gpurun_out/k3f_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 32 -c 1 -o gpurun_out/r02_ncu_attn128 python scripts/forward_probe.py 1 > gpurun_out/k3f_ncu_attn.log 2>&1
