for c in "" "4096:14336:1"; do
  tag=$( [ -z "$c" ] && echo on || echo off )
  WS_GEMM_CHUNKS="$c" WS_PROBE_VERIFY_REQ=32 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gemm_tn --log-file gpurun_out/down_ncu_$tag.csv python scripts/forward_probe.py 1 > gpurun_out/down_ncu_$tag.log 2>&1
done
