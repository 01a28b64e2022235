timeout 300 python scratch/cadence_prof.py > gpurun_out/r2_cad_prof.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cad_launches.csv python scratch/cadence_prof.py > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_cad_launches.csv k_gemm 200 > gpurun_out/r2_cad_launch_sum.txt 2>&1
