mkdir -p gpurun_out/s
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s/gputest.log 2>&1; echo GT $? >> gpurun_out/s/gputest.log
for f in 0 1; do CURVOPT_CG_FUSED=$f timeout 300 python scratch/cgf_diag.py /tmp/cgf$f.npz > /dev/null 2>&1; done
python - > gpurun_out/s/diag.log 2>&1 <<'PY'
import numpy as np
a=np.load('/tmp/cgf0.npz'); b=np.load('/tmp/cgf1.npz')
for k in a.files:
    if k.endswith('_rr'): continue
    print(k, f"{np.linalg.norm(b[k]-a[k])/np.linalg.norm(a[k]):.2e}", a[k+'_rr'], b[k+'_rr'])
PY
timeout 900 python bench.py --no-cpu > gpurun_out/s/bench_c3.log 2>&1
