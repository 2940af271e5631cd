"""Per-block phase timeline of k_assign_qprep on the cfg2 step (variant built with
-DPALS_SCAN_TRACE): PALS_GPU_LIB=_variants/trace.so python scripts/aq_trace.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import _lib, workloads  # noqa: E402
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, Grid, Plan  # noqa: E402

ctx = Context(0)
c = workloads.cfg2()
plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
th, _, _ = plan.scores()
q = workloads.gen_queries(10_000, 2605, float(th.max()), "qos")
d_q = torch.from_numpy(q.view(np.uint8).copy()).cuda()
d_i = torch.empty(len(q), dtype=torch.int32, device="cuda")
d_r = torch.empty(len(q), dtype=torch.uint8, device="cuda")
for _ in range(5):
    plan.run(d_q.data_ptr(), len(q), d_i.data_ptr(), d_r.data_ptr())
torch.cuda.synchronize()
lib = _lib.load()
buf = np.zeros((1024, 8), np.uint64)
lib.pals_debug_aq_trace.argtypes = [C.c_void_p]
assert lib.pals_debug_aq_trace(buf.ctypes.data) == 0
rows = buf.astype(np.int64)
used = rows[:, 0] > 0
t0 = rows[used, 0].min()
r = np.where(rows > 0, rows - t0, -1)
qb = 40  # grid_blocks(1e4 queries, 256): the flat grid's first blocks are qprep
for name, sel in (("assign", np.arange(1024) >= qb), ("qprep", np.arange(1024) < qb)):
    m = used & sel & (rows[:, 7] > 0)
    if not m.any():
        continue
    x = r[m] / 1e3
    print(f"{name}: blocks {m.sum()}")
    for k in (0, 1, 5, 6, 2, 3, 4, 7):
        v = x[:, k]
        v = v[v >= 0]
        if len(v):
            print(f"  mark {k}: min/med/max us {np.percentile(v, [0, 50, 100]).round(2)}")
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
if os.path.isdir(out):
    np.save(os.path.join(out, "aq_trace.npy"), r)
