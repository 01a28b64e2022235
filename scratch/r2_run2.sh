timeout 900 python -m pytest tests/test_gpu_row.py tests/test_gpu_extra.py tests/test_gpu_parity.py -k "row or c4 or cholesky" -x -q -s 2>&1 | tail -30 > gpurun_out/r2_row.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c4b.log 2>&1
