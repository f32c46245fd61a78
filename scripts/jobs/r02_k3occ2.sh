probe() { for n in 107 10 256; do timeout 300 python scripts/k3_probe.py $n 4 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['rows'], round(d['us'],1), round(d['frac'],3))" | tr '\n' ' '; done; echo; }
for rep in 1 2; do
for f in "-DWS_K3_B=4 -DWS_K3_MINB=4" "-DWS_K3_B=8 -DWS_K3_MINB=3" "-DWS_K3_B=8 -DWS_K3_MINB=2" "-DWS_K3_B=6 -DWS_K3_MINB=3"; do
  touch paper_2602_18931_b200/csrc/kernels/rowstats.cu
  NVCC_APPEND_FLAGS="$f" python -c "from paper_2602_18931_b200 import build; build.build()" > /dev/null 2>&1
  echo "[$f] $(probe)" >> gpurun_out/k3occ2.out
done
done
