probe() { for n in 107 256; do timeout 300 python scripts/k3_probe.py $n 4 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['rows'], round(d['us'],1), round(d['frac'],3))"; done; }
for flags in "-DWS_K3_DEC=0" "-DWS_K3_DEC=0 -DWS_K3_MINB=3" "-DWS_K3_DEC=0 -DWS_K3_MINB=4" "-DWS_K3_DEC=1 -DWS_K3_MINB=3" "-DWS_K3_DEC=0 -DWS_K3_RW=8 -DWS_K3_NS=2 -DWS_K3_MINB=4"; do
  touch paper_2602_18931_b200/csrc/kernels/rowstats.cu
  NVCC_APPEND_FLAGS="$flags" python -c "from paper_2602_18931_b200 import build; build.build()" > /dev/null 2>&1
  echo "[$flags] ring" >> gpurun_out/k3v8_probe.log; probe >> gpurun_out/k3v8_probe.log
  echo "[$flags] reg8" >> gpurun_out/k3v8_probe.log; WS_K3_RING=0 probe >> gpurun_out/k3v8_probe.log
  echo "[$flags] reg4" >> gpurun_out/k3v8_probe.log; WS_K3_VW=4 probe >> gpurun_out/k3v8_probe.log
done
for c in 0 1 2 3 4; do
  echo "cfg=$c" >> gpurun_out/attn_sweep.log
  WS_ATTN128=$c WS_PROFILE_MODEL=1 timeout 300 python scripts/forward_probe.py 5 >> gpurun_out/attn_sweep.log 2>&1
done
