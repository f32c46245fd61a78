timeout 600 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
python scripts/forward_probe.py 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_att.csv python scripts/forward_probe.py 1 > /dev/null 2>&1; wc -l gpurun_out/launches_att.csv
