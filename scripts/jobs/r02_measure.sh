python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
WS_PROBE_VERIFY_REQ=107 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_vtraffic.csv python scripts/forward_probe.py 1 > gpurun_out/r02_vtraffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_stats -c 1 -o gpurun_out/r02_ncu_k3_535 python scripts/k3_probe.py 107 4 > gpurun_out/r02_ncu_k3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --launch-skip 60000 --launch-count 1500 --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 1 --warmup 0 > gpurun_out/r02_launches_bench.log 2>&1
ls -la gpurun_out | tail -8
