mkdir -p gpurun_out
python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_ps.py -x -q 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_sliced.json 2>gpurun_out/bench_n2_sliced.err; echo bench rc=$?
