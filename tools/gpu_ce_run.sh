# scratch driver: tests + bench at N=1,2,4
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1d_pytest.log
timeout 900 python bench.py > gpurun_out/r1d_bench_n1.json 2> gpurun_out/r1d_bench_n1.err
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r1d_bench_n$n.json 2> gpurun_out/r1d_bench_n$n.err
done
