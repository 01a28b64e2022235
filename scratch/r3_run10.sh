mkdir -p gpurun_out
CURVOPT_CG_FUSED=0 python scratch/cgf_diag.py /tmp/cgf0.npz > gpurun_out/cgfd.log 2>&1
CURVOPT_CG_FUSED=1 python scratch/cgf_diag.py /tmp/cgf1.npz >> gpurun_out/cgfd.log 2>&1
python - >> gpurun_out/cgfd.log 2>&1 <<'PY'
import numpy as np
a=np.load('/tmp/cgf0.npz'); b=np.load('/tmp/cgf1.npz')
for k in a.files:
    if k.endswith('_rr'): continue
    xa, xb = a[k], b[k]
    print(k, f"{np.linalg.norm(xb-xa)/np.linalg.norm(xa):.2e}", a[k+'_rr'], b[k+'_rr'])
PY
timeout 800 python -m pytest tests/test_gpu_cg_fused.py tests/test_nccl_path.py -x -q > gpurun_out/cgf_test.log 2>&1
