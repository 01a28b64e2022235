timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_gv1024.csv python scratch/gv1024_ncu.py 1024 > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_gv256.csv python scratch/gv1024_ncu.py 256 > /dev/null 2>&1
