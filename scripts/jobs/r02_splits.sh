run() { echo "== $1" >> gpurun_out/splits.out; WS_GEMM_SPLITS="$1" timeout 300 python scripts/gemm_probe.py 7 48,192,496 32,107 2>&1 | grep -o '"model": "[^"]*"\|"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - - >> gpurun_out/splits.out; }
run ""
run "2048:8192:2"
run "2048:8192:4"
run "2048:8192:4,2048:2048:2"
run "2048:8192:4,2048:2048:2,3072:2048:2"
run "4096:14336:2,4096:4096:2"
run ""
