"""Per-step device time (CUDA events) and host time of C3 planned steps (estimator every 10)."""
import sys, time; sys.path.insert(0, ".")
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
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 25):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    w, st, info = meth.step(w, db[i % 4], st)
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"step {i:2d} est={i % 10 == 0} dev {e0.elapsed_time(e1):7.3f} ms host {1e3 * (t1 - t0):7.3f} ms prods {meth.last_products}")
