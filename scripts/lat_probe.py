"""Where the single-call latency goes: empty launch+sync, tiny H2D/D2H round trips,
pals_select_one / pals_control_step_one on cfg1 (36 candidates)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import workloads  # noqa: E402
from paper_2605_21427_b200.wattserve import (AnalyticModel, Context, Grid, Plan,  # noqa: E402
                                             make_targets, select_config)


def t(fn, n=300):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


x = torch.zeros(16, device="cuda")
h = torch.zeros(256, dtype=torch.uint8).pin_memory()
d = torch.zeros(256, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
print("empty kernel + sync us", t(lambda: (x.add_(1), torch.cuda.synchronize())))
print("H2D 256B + sync us", t(lambda: (d.copy_(h, non_blocking=True), torch.cuda.synchronize())))
print("H2D + kernel + D2H + sync us",
      t(lambda: (d.copy_(h, non_blocking=True), d.add_(1), h.copy_(d, non_blocking=True),
                 torch.cuda.synchronize())))
ctx = Context(0)
c1 = workloads.cfg1()
m1 = AnalyticModel(ctx, c1["profile"], c1["gpu"])
th, _, _ = Plan(m1, Grid(ctx, c1["points"]), c1["coeffs"]).scores()
tg = make_targets(0.6 * float(th.max()), 1600.0)
print("select_config us", t(lambda: select_config(c1["points"], tg, m1, c1["coeffs"], 1.0, 0.05, 0.02)))
