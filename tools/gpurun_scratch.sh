mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
( time timeout 900 python bench.py > gpurun_out/fin_bench_n1.json 2>gpurun_out/fin_bench_n1.err ) 2>&1 | grep real
for n in 2 4; do
( time timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n > gpurun_out/fin_bench_n$n.json 2>gpurun_out/fin_bench_n$n.err ) 2>&1 | grep real
done
( time timeout 600 python bench.py --impl reference > gpurun_out/fin_bench_ref.json 2>/dev/null ) 2>&1 | grep real
( time timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29599 bench.py --impl reference --gpus 2 > gpurun_out/fin_bench_ref_n2.json 2>/dev/null ) 2>&1 | grep real
