set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2_gputest.log
timeout 600 python bench.py > gpurun_out/r2_bench_c3.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c5.log 2>&1
tail -3 gpurun_out/*.log
