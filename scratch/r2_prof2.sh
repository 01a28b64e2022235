timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_c3_launches.csv > gpurun_out/r2_c3_launch_sum.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cad_launches.csv python scratch/cadence_prof.py > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_cad_launches.csv > gpurun_out/r2_cad_launch_sum.txt 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python scratch/c4_ncu.py > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_c4_launches.csv > gpurun_out/r2_c4_launch_sum.txt 2>&1
timeout 300 python scratch/small_gv.py > gpurun_out/r2_small_gv.log 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench_c3_final.log 2>&1
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/r2_bench_c4_final.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r2_bench_c5_final.log 2>&1
timeout 600 python bench.py --config cadence --steps 300 --warmup 3 > gpurun_out/r2_bench_cad_final.log 2>&1
