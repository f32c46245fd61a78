timeout 900 python -m pytest tests/test_gpu_rowstats.py tests/test_gpu_sample.py -x -q -m gpu > gpurun_out/k3v4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k3v4_tests.log
for n in 107 10 256; do timeout 300 python scripts/k3_probe.py $n 4 >> gpurun_out/k3v4_probe.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stats -c 1 -o gpurun_out/r02_ncu_k3v4_535 python scripts/k3_probe.py 107 4 > gpurun_out/k3v4_ncu.log 2>&1
for mb in 3 4; do
  touch paper_2602_18931_b200/csrc/kernels/rowstats.cu
  NVCC_APPEND_FLAGS="-DWS_K3_MINB=$mb" python -c "from paper_2602_18931_b200 import build; build.build()" > /dev/null 2>&1
  echo "minb=$mb" >> gpurun_out/k3v4_probe.log
  for n in 107 10 256; do timeout 300 python scripts/k3_probe.py $n 4 >> gpurun_out/k3v4_probe.log 2>&1; done
done
