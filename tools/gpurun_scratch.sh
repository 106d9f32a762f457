# scratch command file for one gpurun call (rewritten per experiment)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/exce_probe.py > gpurun_out/exce2.log 2>&1
