timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python scratch/c4_ncu.py > gpurun_out/r2_c4_ncu.log 2>&1
python scratch/launch_sum.py gpurun_out/r2_c4_launches.csv k_gemm_tc2 14 > gpurun_out/r2_c4_launch_sum.txt 2>&1
