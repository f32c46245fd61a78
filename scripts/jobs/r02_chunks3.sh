run() { echo "== $1" >> gpurun_out/chunks3.out; WS_GEMM_CHUNKS="$1" timeout 300 python scripts/gemm_probe.py 7 48,116,256,496 32,64,107 2>&1 | grep -o '"model": "[^"]*"\|"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - - >> gpurun_out/chunks3.out; }
run ""
run "2048:2048:2"
run "4096:4096:2"
run "2048:2048:2,4096:4096:2,16384:2048:2,28672:4096:2"
run ""
