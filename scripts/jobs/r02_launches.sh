timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --launch-skip 600 --launch-count 3000 --log-file gpurun_out/r02_launches_bench16.csv python bench.py --requests 16 --steps 1 --warmup 0 > gpurun_out/r02_launches_bench16.log 2>&1
echo "rc=$?" >> gpurun_out/r02_launches_bench16.log
