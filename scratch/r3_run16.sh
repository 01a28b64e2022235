mkdir -p gpurun_out/u
timeout 900 python -m pytest tests/test_gpu_cg_fused.py tests/test_gpu_gates.py tests/test_gpu_parity.py tests/test_nccl_path.py -q -m gpu > gpurun_out/u/t.log 2>&1; echo GT $? >> gpurun_out/u/t.log
timeout 900 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/u/bench_c3.log 2>&1
