timeout 2000 python -m pytest tests -x -q -m gpu > gpurun_out/fs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fs_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/fs_n1.json 2> gpurun_out/fs_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/fs_n2.json 2> gpurun_out/fs_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/fs_n4.json 2> gpurun_out/fs_n4.err
