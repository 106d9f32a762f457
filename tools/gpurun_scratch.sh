# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python bench.py --no-cpu --no-sweep --no-ps > gpurun_out/aff_n1.json 2> gpurun_out/aff_n1.err
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-cpu --no-sweep --no-ps > gpurun_out/aff_n$n.json 2> gpurun_out/aff_n$n.err
done
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
