for n in 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r1e_bench_n$n.json 2> gpurun_out/r1e_bench_n$n.err
done
