mkdir -p gpurun_out
for f in 0 1; do echo "FUSED=$f"; CURVOPT_CG_FUSED=$f timeout 300 python scratch/cgf_oracle.py; done > gpurun_out/cgfo.log 2>&1
