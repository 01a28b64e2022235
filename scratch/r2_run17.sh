timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2_gputest.log
timeout 300 python scratch/cadence_prof.py > gpurun_out/r2_cad_prof.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cad_launches.csv python scratch/cadence_prof.py > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_cad_launches.csv k_gemm 200 > gpurun_out/r2_cad_launch_sum.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1
