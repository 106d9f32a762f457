mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ring_rounds tools/k1v/ring_rounds.cu && timeout 300 /tmp/ring_rounds | tee gpurun_out/ring_rounds.jsonl
