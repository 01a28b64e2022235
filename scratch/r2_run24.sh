timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_pipeline.py tests/test_harness.py -q -x 2>&1 | tail -15 > gpurun_out/r2_graphs.log
timeout 600 python bench.py --steps 50 --warmup 10 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1
timeout 600 python bench.py --config cadence --steps 300 --warmup 3 --no-cpu > gpurun_out/r2_bench_cadence.log 2>&1
