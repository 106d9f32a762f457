mkdir -p gpurun_out
( time timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 bench.py --gpus 4 > gpurun_out/fin2_bench_n4.json 2>gpurun_out/fin2_bench_n4.err ) 2>&1 | grep real
