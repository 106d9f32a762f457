mkdir -p gpurun_out
for n in 2 4; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n > gpurun_out/r1s_bench_n$n.json 2>gpurun_out/r1s_bench_n$n.err; echo bench $n rc=$?
done
