timeout 300 python scratch/rowcg_diag.py > gpurun_out/r2_rowcg_diag.log 2>&1
CURVOPT_PDL=0 timeout 600 python scratch/c4_prof.py > gpurun_out/r2_c4_prof.log 2>&1
