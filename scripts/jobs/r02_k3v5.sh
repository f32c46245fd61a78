timeout 900 python -m pytest tests/test_gpu_rowstats.py tests/test_gpu_sample.py -x -q -m gpu > gpurun_out/k3v5_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k3v5_tests.log
probe() { for n in 107 10 256; do timeout 300 python scripts/k3_probe.py $n 4 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['rows'], round(d['us'],1), round(d['frac'],3))"; done; }
echo "minb=1 vw=8" >> gpurun_out/k3v5_probe.log; probe >> gpurun_out/k3v5_probe.log
echo "minb=1 vw=4" >> gpurun_out/k3v5_probe.log; WS_K3_VW=4 probe >> gpurun_out/k3v5_probe.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stats -c 1 -o gpurun_out/r02_ncu_k3v5_535 python scripts/k3_probe.py 107 4 > gpurun_out/k3v5_ncu.log 2>&1
for mb in 3 4; do
  touch paper_2602_18931_b200/csrc/kernels/rowstats.cu
  NVCC_APPEND_FLAGS="-DWS_K3_MINB=$mb" python -c "from paper_2602_18931_b200 import build; build.build()" > /dev/null 2>&1
  echo "minb=$mb vw=8" >> gpurun_out/k3v5_probe.log; probe >> gpurun_out/k3v5_probe.log
  echo "minb=$mb vw=4" >> gpurun_out/k3v5_probe.log; WS_K3_VW=4 probe >> gpurun_out/k3v5_probe.log
done
