"""cProfile of C3 planned steps: where the host spends its time between launches."""
import sys, cProfile, pstats; sys.path.insert(0, ".")
import torch
import bench
import paper_2603_25976_b200 as P
dev = torch.device("cuda", 0)
model = P.Model(bench.DIMS[0], bench.DIMS[1:-1], bench.DIMS[-1], "relu")
meth = P.assemble(bench.spec_c3(), model)
w = P.init_params(model, P.Rng(0)).to_device(dev)
hb = bench.make_batches(4, bench.GLOBAL_B, 0, 1)
db = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=bench.GLOBAL_B) for X, y in hb]
st = meth.init(w, 0)
for i in range(5):
    w, st, info = meth.step(w, db[i % 4], st)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(20):
    w, st, info = meth.step(w, db[i % 4], st)
pr.disable()
ps = pstats.Stats(pr).sort_stats("tottime")
ps.print_stats(18)
