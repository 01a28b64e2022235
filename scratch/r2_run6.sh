timeout 900 python -m pytest tests/test_gpu_row.py tests/test_gpu_extra.py -q 2>&1 | tail -3 > gpurun_out/r2_row.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python scratch/c4_ncu.py > gpurun_out/r2_c4_ncu.log 2>&1
python scratch/launch_sum.py gpurun_out/r2_c4_launches.csv k_gemm_tc2 30 > gpurun_out/r2_c4_launch_sum.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_potrf_diag --launch-skip 20 -c 1 -o gpurun_out/r2_potrf -f python scratch/c4_ncu.py > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_gemm_tc2 --launch-skip 12 -c 1 -o gpurun_out/r2_trail -f python scratch/c4_ncu.py > /dev/null 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c4b.log 2>&1
