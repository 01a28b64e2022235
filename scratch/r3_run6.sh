mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_cg_fused -c 12 --csv --log-file gpurun_out/cgk.csv python scratch/cg_fused_check.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cg_fused -s 4 -c 1 -o gpurun_out/cgf2 python scratch/cg_fused_check.py > gpurun_out/ncu_cgf.log 2>&1
