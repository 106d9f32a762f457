# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1h_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1h_pytest.log
timeout 900 python bench.py --no-cpu --no-sweep > gpurun_out/r1h_bench_n1.json 2> gpurun_out/r1h_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-cpu --no-sweep > gpurun_out/r1h_bench_n2.json 2> gpurun_out/r1h_bench_n2.err
