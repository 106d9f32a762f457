# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1q_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1q_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r1q_pytest.log 2>&1
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/r1q_bench_n1.json 2> gpurun_out/r1q_bench_n1.err; echo "n1 $(( $(date +%s) - s )) s" > gpurun_out/r1q_times.txt
for n in 2 4; do
s=$(date +%s); timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r1q_bench_n$n.json 2> gpurun_out/r1q_bench_n$n.err; echo "n$n $(( $(date +%s) - s )) s" >> gpurun_out/r1q_times.txt
done
timeout 600 python bench.py --impl reference > gpurun_out/r1q_ref_n1.json 2> gpurun_out/r1q_ref_n1.err
