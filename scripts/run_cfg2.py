"""Minimal cfg2 step loop (plan.run) for profiler captures."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import workloads  # noqa: E402
from paper_2605_21427_b200.abi import QUERY_DT  # noqa: E402
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, Grid, Plan  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ctx = Context(0)
c = workloads.cfg2(10_000)
plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
th, _, _ = plan.scores()
q = workloads.gen_queries(10_000, c["seed"], float(th.max()), "qos")
dq = torch.from_numpy(np.ascontiguousarray(q, QUERY_DT).view(np.uint8)).cuda()
di = torch.empty(len(q), dtype=torch.int32, device="cuda")
dr = torch.empty(len(q), dtype=torch.uint8, device="cuda")
for _ in range(steps):
    plan.run(dq.data_ptr(), len(q), di.data_ptr(), dr.data_ptr())
torch.cuda.synchronize()
print("ok", int(di.cpu().numpy().sum()))
