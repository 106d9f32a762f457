# scratch command file for one gpurun call (rewritten per experiment)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/al2_pytest.log 2>&1; echo rc=$? >> gpurun_out/al2_pytest.log
timeout 300 python tools/align_probe.py inproc > gpurun_out/align4.log 2>&1
timeout 600 python bench.py --no-cpu --no-ps --no-sweep > gpurun_out/al2_n1.json 2> gpurun_out/al2_n1.err
