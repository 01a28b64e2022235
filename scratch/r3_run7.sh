mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cg_fused -c 12 --csv --log-file gpurun_out/cgk.csv python scratch/cg_fused_check.py > /dev/null 2>&1
for f in 1 0 1; do echo "FUSED=$f"; CURVOPT_CG_FUSED=$f timeout 300 python scratch/cg_iter_time.py; done > gpurun_out/cgit.log 2>&1
timeout 600 python -m pytest tests/test_nccl_path.py -x -q > gpurun_out/gt.log 2>&1; echo GT $? >> gpurun_out/gt.log
