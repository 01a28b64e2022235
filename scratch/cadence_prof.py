"""One newton_cg step of the cadence workload (rho off) inside cudaProfilerStart/Stop,
plus wall vs device time of 50 steps."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_25976_b200._lib as L
if len(sys.argv) > 1: L.LIB_PATH = sys.argv[1]
import paper_2603_25976_b200 as P
from paper_2603_25976_b200 import harness as H
tr, _ = H.gen_regression(20000, 512, 0.1, 0)
model = P.Model(512, (1024, 1024), 1, "relu")
meth = H.cadence_methods([-1], model)[-1]
root = P.Rng(0)
w = P.init_params(model, root.split()).to_device()
bat = H.EpochBatcher(tr, 256, root.split())
st = meth.init(w, seed=0)
bs = [bat.next() for _ in range(8)]
for i in range(20):
    w, st, info = meth.step(w, bs[i % 8], st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for i in range(50):
    w, st, info = meth.step(w, bs[i % 8], st)
e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"50 steps: wall {1e3*(t1-t0)/50:.3f} ms/step, events {e0.elapsed_time(e1)/50:.3f} ms/step, info {info}")
torch.cuda.cudart().cudaProfilerStart()
w, st, info = meth.step(w, bs[0], st); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
