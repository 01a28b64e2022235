timeout 900 python -m pytest tests/test_gpu_row.py tests/test_gpu_extra.py tests/test_gpu_parity.py -k "row or c4 or cholesky or not_pd" -q -x 2>&1 | tail -3 > gpurun_out/r2_row.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches_b.csv python scratch/c4_ncu.py > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_c4_launches_b.csv > gpurun_out/r2_c4_launch_sum_b.txt 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c4b.log 2>&1
