"""Per-CTA phase timeline of k_scan (variant built with -DPALS_SCAN_TRACE):
PALS_GPU_LIB=_variants/trace.so python scripts/scan_trace.py [cfg2|cfg3]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import _lib, workloads  # noqa: E402
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, Grid, Plan  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
ctx = Context(0)
c = workloads.cfg2() if which == "cfg2" else workloads.cfg3()
plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
th, _, _ = plan.scores()
nq = 10_000 if which == "cfg2" else 1_000_000
q = (workloads.gen_queries(nq, 2605, float(th.max()), "qos") if which == "cfg2" else
     workloads.gen_queries(nq, 2605, float(th.max()), "mixed", budget=(600.0, 2000.0)))
d_q = torch.from_numpy(q.view(np.uint8).copy()).cuda()
d_i = torch.empty(nq, dtype=torch.int32, device="cuda")
d_r = torch.empty(nq, dtype=torch.uint8, device="cuda")
plan.time_scan(True)
for _ in range(5):
    plan.run(d_q.data_ptr(), nq, d_i.data_ptr(), d_r.data_ptr())
torch.cuda.synchronize()
lib = _lib.load()
buf = np.zeros((4096, 16), np.uint64)
lib.pals_debug_scan_trace.argtypes = [C.c_void_p, C.c_int]
assert lib.pals_debug_scan_trace(buf.ctypes.data, 4096) == 0
rows = buf[(buf[:, 0] > 0) & (buf[:, 15] > 0)].astype(np.int64)
t0 = rows[:, 0].min()
print(f"CTAs {len(rows)}  scan_ms {plan.scan_ms():.4f}")
print("start  : min/med/max us", np.percentile((rows[:, 0] - t0) / 1e3, [0, 50, 100]).round(2))
print("end    : min/med/max us", np.percentile((rows[:, 15] - t0) / 1e3, [0, 50, 100]).round(2))
for k in range(1, 15):
    m = rows[:, k] > 0
    if not m.any():
        continue
    prev = rows[:, k - 1]
    d = (rows[m, k] - prev[m]) / 1e3
    print(f"mark {k:2d} (n={m.sum():4d}) dt min/med/max us", np.percentile(d, [0, 50, 100]).round(2))
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
if os.path.isdir(out):
    np.save(os.path.join(out, f"scan_trace_{which}.npy"), rows - t0)
