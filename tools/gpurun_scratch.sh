mkdir -p gpurun_out
timeout 900 python bench.py --no-ps > gpurun_out/geo_n1b.json 2>/dev/null; echo rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --no-ps --no-cpu > gpurun_out/geo_n2b.json 2>/dev/null; echo rc=$?
SRFLOW_CTAS_PER_SM=2 SRFLOW_COPY_THREADS=256 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --no-ps --no-cpu > gpurun_out/geo_n2old.json 2>/dev/null; echo rc=$?
SRFLOW_CTAS_PER_SM=2 SRFLOW_COPY_THREADS=256 timeout 900 python bench.py --no-ps > gpurun_out/geo_n1old.json 2>/dev/null; echo rc=$?
