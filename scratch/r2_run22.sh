timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r2_gputest.log
timeout 600 python bench.py --config cadence --steps 300 --warmup 3 --no-cpu > gpurun_out/r2_bench_cadence.log 2>&1
