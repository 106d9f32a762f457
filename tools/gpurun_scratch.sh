mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-sweep > gpurun_out/ord_n1.json 2>/dev/null; echo rc=$?
for n in 2 4; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --no-sweep > gpurun_out/ord_n$n.json 2>/dev/null; echo rc$n=$?
done
