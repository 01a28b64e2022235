timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2_gputest.log
timeout 300 python scratch/small_gv.py > gpurun_out/r2_small_gv.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_gv8192.csv python scratch/gv1024_ncu.py 8192 > /dev/null 2>&1
timeout 600 python bench.py --steps 50 --warmup 10 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1
