# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests/test_gpu_ps.py -x -q > gpurun_out/r1j_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1j_pytest.log
timeout 900 python bench.py --no-cpu --no-sweep > gpurun_out/r1j_bench_n1.json 2> gpurun_out/r1j_bench_n1.err
