timeout 600 python -m pytest tests/test_gpu_gates.py -k "tensor_core_primitives" -q 2>&1 | grep -E "assert|Error|passed|failed|where" | head -30 > gpurun_out/r2_tcprim.log
timeout 300 python scratch/cadence_prof.py > gpurun_out/r2_cad_prof.log 2>&1
