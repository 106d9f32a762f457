mkdir -p gpurun_out
for n in 2 4; do
for lane in 96 128 192; do
  for cfg in "8 static 16" "4 static 16" "8 static 0"; do
    set -- $cfg
    part=""; [ "$3" != "0" ] && part="$3"
    SRFLOW_PS_PUSH_CTAS=$lane PROBE_PARTITION=$part PROBE_SLICES=$1 PROBE_GRAD=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 tools/ps_slice_probe.py 2>>gpurun_out/r2s_ps_lane4.err | grep '^{' | sed "s/^/{\"lane\": $lane, \"partition\": \"$3\", \"r\": /; s/\$/}/" >> gpurun_out/r2s_ps_lane4.jsonl
  done
done
done
echo done
