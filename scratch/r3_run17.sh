mkdir -p gpurun_out/w
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cg_(fused|start)" -s 2 -c 3 -o /tmp/cgfull python scratch/cg_fused_check.py > gpurun_out/w/ncu.log 2>&1
ncu -i /tmp/cgfull.ncu-rep --page details --csv > gpurun_out/w/details.csv 2>/dev/null
