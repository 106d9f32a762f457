mkdir -p gpurun_out
for n in 2 4; do
PROBE_GRAD=static PROBE_SLICES=0,4,2,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 tools/ps_slice_probe.py 2>gpurun_out/slice_err_$n.log | grep '^{' >> gpurun_out/slice_probe3.jsonl
PROBE_GRAD=static PROBE_PARTITION=16 PROBE_SLICES=0,4 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 tools/ps_slice_probe.py 2>>gpurun_out/slice_err_$n.log | grep '^{' | sed 's/^{/{"partition": 16, /' >> gpurun_out/slice_probe3.jsonl
done
