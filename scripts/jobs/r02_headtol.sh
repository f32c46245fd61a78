for c in "" "2048:8192:1"; do
  echo "== chunks rule [$c]" >> gpurun_out/headtol.log
  WS_GEMM_CHUNKS="$c" WS_STAGE_TOL=1 timeout 900 python -m pytest tests/test_gpu_model_parity.py -k real_shapes -q -s -m gpu 2>&1 | grep -E "worst|passed|failed" >> gpurun_out/headtol.log
done
