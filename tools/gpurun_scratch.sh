# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests/test_gpu_ps.py tests/test_gpu_multiprocess.py -x -q > gpurun_out/pw_pytest.log 2>&1; echo rc=$? >> gpurun_out/pw_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for cfg in vgg fcn5 lstm; do
for m in exchange exchange_pw; do
PROBE_CFG=$cfg PROBE_MODE=$m timeout 300 $TR tools/ps_phase_probe.py >> gpurun_out/pw_probe.log 2>&1
done; done
