mkdir -p gpurun_out
for n in 2 4; do
for cfg in fcn5 lstm; do
for g in dynamic static; do
PROBE_CFG=$cfg PROBE_GRAD=$g PROBE_SLICES=0,4,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 tools/ps_slice_probe.py 2>>gpurun_out/slice_err.log | grep '^{' >> gpurun_out/slice_probe4.jsonl
done; done; done
