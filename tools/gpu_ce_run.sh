TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for cfg in lstm fcn5; do
for m in ce phases; do
PROBE_HOST=1 PROBE_CFG=$cfg PROBE_MODE=$m timeout 300 $TR tools/ps_phase_probe.py >> gpurun_out/dbg_ce12.log 2>&1
done; done
