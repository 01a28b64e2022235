timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2_gputest.log
timeout 300 python scratch/small_gv.py > gpurun_out/r2_small_gv.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_gv256b.csv python scratch/gv1024_ncu.py 256 > /dev/null 2>&1
timeout 600 python bench.py --config cadence --steps 300 --warmup 3 --no-cpu > gpurun_out/r2_bench_cadence.log 2>&1
