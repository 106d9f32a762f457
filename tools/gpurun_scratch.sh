# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/dyn_pytest.log 2>&1; echo rc=$? >> gpurun_out/dyn_pytest.log
python -c "
import sys; sys.path.insert(0, '.')
import bench, json
for s in (1024, 1<<20, 16<<20, 256<<20):
    print(s, json.dumps(bench.dynamic_device_rate(s, 0)), flush=True)
" > gpurun_out/dyn_dev.log 2>&1
