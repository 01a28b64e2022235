"""Host-time breakdown of the step boundary on graph steps: sync return -> _finalize return ->
step() entry -> StepGraph.replay entry -> graph launch call (C3)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2603_25976_b200 as P
import paper_2603_25976_b200.method as M
marks = []
pc = time.perf_counter
orig_cpu = torch.Tensor.cpu
def cpu(self, *a, **k):
    r = orig_cpu(self, *a, **k); marks.append(("sync", pc())); return r
torch.Tensor.cpu = cpu
orig_fin = M.Method._finalize
def fin(self, *a, **k):
    r = orig_fin(self, *a, **k); marks.append(("fin_ret", pc())); return r
M.Method._finalize = fin
orig_step = M.Method.step
def step(self, *a, **k):
    marks.append(("step_in", pc())); return orig_step(self, *a, **k)
M.Method.step = step
orig_rep = M.StepGraph.replay
def rep(self, *a, **k):
    marks.append(("replay_in", pc())); return orig_rep(self, *a, **k)
M.StepGraph.replay = rep
orig_gr = torch.cuda.CUDAGraph.replay
def gr(self):
    marks.append(("launch", pc())); orig_gr(self)
torch.cuda.CUDAGraph.replay = gr
dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(25):
    w, st, info = meth.step(w, db[i % 4], st)
marks.clear()
for i in range(40):
    w, st, info = meth.step(w, db[i % 4], st)
seq = ["sync", "fin_ret", "step_in", "replay_in", "launch"]
d = {k: [] for k in seq[1:]}
cur = {}
for k, t in marks:
    if k == "sync": cur = {"sync": t}
    elif k in seq and cur:
        cur[k] = t
        if k == "launch" and all(s in cur for s in seq):
            for a, b in zip(seq, seq[1:]): d[b].append((cur[b] - cur[a]) * 1e6)
            cur = {}
for k in seq[1:]: print(f"-> {k:10s} median {np.median(d[k]):6.1f} us (n={len(d[k])})")
