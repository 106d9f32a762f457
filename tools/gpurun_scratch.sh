# scratch command file for one gpurun call (rewritten per experiment)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for kib in 0 131072 32768; do
SRFLOW_PEER_CE_KIB=$kib timeout 900 $TR bench.py --gpus 2 --no-cpu --no-ps --steps 10 > gpurun_out/al_n2_$kib.json 2> gpurun_out/al_n2_$kib.err
done
