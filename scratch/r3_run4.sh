mkdir -p gpurun_out
for f in "CURVOPT_CG_FUSED=0" "CURVOPT_CG_FUSED=1" "CURVOPT_CG_FUSED=0" "CURVOPT_CG_FUSED=1"; do env $f timeout 300 python scratch/phase_time.py >> gpurun_out/phase_$f.log 2>&1; done
for f in 0 1; do CURVOPT_CG_FUSED=$f timeout 300 python scratch/cg_fused_check.py > gpurun_out/hash_$f.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cg -c 40 --csv --log-file gpurun_out/cgk.csv python scratch/cg_fused_check.py > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; echo GT $? >> gpurun_out/gt.log
