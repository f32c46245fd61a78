for c in 0 1 2 3 4; do
  echo "cfg=$c" >> gpurun_out/attn_sweep.log
  WS_ATTN128=$c WS_PROFILE_MODEL=1 timeout 300 python scripts/forward_probe.py 5 >> gpurun_out/attn_sweep.log 2>&1
done
