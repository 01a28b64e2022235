timeout 300 python scratch/cadence_prof.py scratch/libA.so > gpurun_out/r2_cadA.log 2>&1
timeout 300 python scratch/cadence_prof.py scratch/libB.so > gpurun_out/r2_cadB.log 2>&1
