mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-ps > /dev/null 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 300 --csv --log-file gpurun_out/launches_n1_r1g.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-ps > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
