"""5 C3 planned steps; prints a hash of the final weights and the StepInfo rows (compare CURVOPT_CG_SPLIT_FUSED=0/1)."""
import sys, hashlib; sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(12):
    w, st, info = meth.step(w, db[i % 4], st)
    print(i, info.solver_iterations, info.solver_converged, f"{info.loss_before:.9f}", f"{info.step_norm:.9e}")
print("hash", hashlib.sha256(w.data.cpu().numpy().tobytes()).hexdigest()[:16])
