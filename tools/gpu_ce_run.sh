set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/ce_kern.log 2>&1; echo rc=$? >> gpurun_out/ce_kern.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
SRFLOW_PEER_CE_KIB=0 timeout 300 $TR tools/ring_probe.py > gpurun_out/ce_ring_sm.log 2>&1
timeout 300 $TR tools/ring_probe.py > gpurun_out/ce_ring_ce.log 2>&1
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/ce_bench_n2.json 2> gpurun_out/ce_bench_n2.err
