timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2_gputest.log
timeout 300 python scratch/small_gv.py > gpurun_out/r2_small_gv.log 2>&1
timeout 300 python scratch/headdiag.py > gpurun_out/r2_headdiag.log 2>&1
timeout 600 python bench.py --config cadence --steps 300 --warmup 3 --no-cpu > gpurun_out/r2_bench_cadence.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1
