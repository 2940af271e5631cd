"""Quick GPU timing of the cfg2 / cfg3 select step and its pair-scan kernel, with a parity
check against the C oracle on a query sample:  python scripts/select_quick.py [cfg2|cfg3] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import workloads  # noqa: E402
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, Grid, Plan  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
c = workloads.cfg2() if which == "cfg2" else workloads.cfg3()
plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
th, _, _ = plan.scores()
nq = 10_000 if which == "cfg2" else 1_000_000
q = (workloads.gen_queries(nq, 2605, float(th.max()), "qos") if which == "cfg2" else
     workloads.gen_queries(nq, 2605, float(th.max()), "mixed", budget=(600.0, 2000.0)))
d_q = torch.from_numpy(q.view(np.uint8).copy()).cuda()
d_i = torch.empty(nq, dtype=torch.int32, device="cuda")
d_r = torch.empty(nq, dtype=torch.uint8, device="cuda")
# "graph": time the captured step with its PDL edges (no scan events in the graph)
graph_only = len(sys.argv) > 4 and sys.argv[4] == "graph"
plan.time_scan(not graph_only)
run = lambda: plan.run(d_q.data_ptr(), nq, d_i.data_ptr(), d_r.data_ptr())  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
st = plan.stats()
pairs = int(st[0] + st[1] + st[2]) * len(c["points"])
scan, step = [], []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run()
    e1.record(stream)
    torch.cuda.synchronize()
    step.append(e0.elapsed_time(e1))
    scan.append(plan.scan_ms() if not graph_only else float("nan"))
ms = float(np.median(scan))
print(f"{which}: pairs {pairs:.4g}  scan {ms * 1e3:.1f} us ({pairs / (ms * 1e-3):.4g} pairs/s)  "
      f"step {np.median(step) * 1e3:.1f} us ({pairs / (np.median(step) * 1e-3):.4g} pairs/s)")
idx = d_i.cpu().numpy()
rs = d_r.cpu().numpy()
if len(sys.argv) < 4:
    from oracle.oracle import Oracle
    orc = Oracle()
    T, P, _ = orc.eval(c["profile"], c["gpu"], c["points"])
    sub = np.arange(0, nq, max(1, nq // 400))
    oi, orr, _ = orc.select(c["points"], T, P, c["coeffs"], q[sub])
    print("parity sample", len(sub), "ok" if np.array_equal(idx[sub], oi) and
          np.array_equal(rs[sub], orr) else "MISMATCH")
