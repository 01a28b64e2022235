mkdir -p gpurun_out/p
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_harness.py tests/test_host_api.py -q -m gpu > gpurun_out/p/t.log 2>&1; echo GT $? >> gpurun_out/p/t.log
timeout 900 python bench.py --no-cpu > gpurun_out/p/bench_c3.log 2>&1
timeout 900 python bench.py --config cadence --steps 300 --warmup 3 > gpurun_out/p/bench_cad.log 2>&1
