# scratch command file for one gpurun call (rewritten per experiment)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
timeout 300 $TR tools/ps_phase_probe.py >> gpurun_out/ap.log 2>&1
PROBE_CFG=fcn5 timeout 300 $TR tools/ps_phase_probe.py >> gpurun_out/ap.log 2>&1
timeout 300 python tools/ps_profile.py vgg phases >> gpurun_out/ap.log 2>&1
