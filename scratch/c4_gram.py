"""Build the C4 row-lane Gram once (snapshot + cv_row_gram) at batch b: for ncu captures of the Gram GEMMs."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200 as P
b = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
m = P.Model(3072, (2048, 2048), 10, "relu")
w = P.init_params(m, P.Rng(0)).to_device()
r = P.Rng(1)
X = torch.from_numpy(r.normal(b * 3072).reshape(b, 3072).astype(np.float32)).cuda()
y = torch.from_numpy(r.integers(b, 10)).cuda()
snap = P.make_snapshot("ggn_ce", m, w, P.Batch(X, y, "ce"))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
G = snap.row.gram()
e1.record(); torch.cuda.synchronize()
mm = b * 10
fl = sum(2.0 * mm * mm * k for k in (2048, 2048, 10))
print(f"gram m={mm}: {e0.elapsed_time(e1):.2f} ms incl. seeds; SYRK-equivalent {fl / 2 / 1e12:.2f} TFLOP useful")
