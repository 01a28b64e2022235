mkdir -p gpurun_out
timeout 800 python -m pytest tests/test_gpu_cg_fused.py tests/test_nccl_path.py tests/test_gpu_gates.py -x -q > gpurun_out/cgf_test.log 2>&1
