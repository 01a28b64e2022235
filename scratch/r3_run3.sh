mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cg_fused -s 4 -c 1 -o gpurun_out/cgf python scratch/cg_fused_check.py > gpurun_out/ncu_cgf.log 2>&1
