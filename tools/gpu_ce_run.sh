# scratch driver for gpurun experiments (copy-engine paths)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/ce_pytest.log 2>&1; echo rc=$? >> gpurun_out/ce_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for kib in 0 1024 16384; do
SRFLOW_PEER_CE_KIB=$kib timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/ce_bench_n2_$kib.json 2> gpurun_out/ce_bench_n2_$kib.err
done
