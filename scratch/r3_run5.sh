mkdir -p gpurun_out
for f in 0 1 0 1; do echo "FUSED=$f"; CURVOPT_CG_FUSED=$f timeout 300 python scratch/cg_iter_time.py; done > gpurun_out/cgit.log 2>&1
timeout 600 python -m pytest tests/test_nccl_path.py -x -q > gpurun_out/gt.log 2>&1; echo GT $? >> gpurun_out/gt.log
