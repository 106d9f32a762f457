mkdir -p gpurun_out
for lane in 112 128 144; do
  for cfg in "4 static" "8 static" "16 static"; do
    set -- $cfg
    SRFLOW_PS_PUSH_CTAS=$lane PROBE_SLICES=$1 PROBE_GRAD=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/ps_slice_probe.py 2>>gpurun_out/r2s_ps_lane3.err | grep '^{' | sed "s/^/{\"lane\": $lane, \"r\": /; s/\$/}/" >> gpurun_out/r2s_ps_lane3.jsonl
  done
done
echo done
