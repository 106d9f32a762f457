# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests/test_gpu_ps.py -x -q > gpurun_out/lb_pytest.log 2>&1; echo rc=$? >> gpurun_out/lb_pytest.log
timeout 900 python bench.py --no-cpu --no-sweep > gpurun_out/lb_n1.json 2> gpurun_out/lb_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-cpu --no-sweep > gpurun_out/lb_n2.json 2> gpurun_out/lb_n2.err
