"""Time pals_plan_frontier (host output) call by call on the cfg3x grid."""
import time

import torch

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, Grid, Plan

ctx = Context(0)
c = workloads.cfg3_extended()
plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
n = len(c["points"])
d_idx = torch.empty(n, dtype=torch.int32, device="cuda")
d_n = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.frontier_device(d_idx.data_ptr(), d_n.data_ptr())
torch.cuda.synchronize()
for k in range(6):
    t0 = time.perf_counter()
    idx = plan.frontier()
    print(f"call {k}: {1e3 * (time.perf_counter() - t0):.3f} ms, {len(idx)} points")
for k in range(3):
    t0 = time.perf_counter()
    plan.prepare()
    torch.cuda.synchronize()
    print(f"prepare {k}: {1e3 * (time.perf_counter() - t0):.3f} ms")
