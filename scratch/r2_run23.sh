timeout 600 python -m pytest tests/test_gpu_pipeline.py -q 2>&1 | tail -3 > gpurun_out/r2_pipe.log
timeout 600 python bench.py --steps 50 --warmup 10 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1
