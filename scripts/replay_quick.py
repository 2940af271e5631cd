"""Quick GPU timing of the cfg4 replay (synthetic thread / warp layouts and the caller-trace
path) with a parity check of the three against each other:
  python scripts/replay_quick.py [n_traces] [n_steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import workloads  # noqa: E402
from paper_2605_21427_b200.abi import SUMMARY_DT, TraceBatch  # noqa: E402
from paper_2605_21427_b200.wattserve import (AnalyticModel, Context, replay_device,  # noqa: E402
                                             replay_traces_device)

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 3600
ctx = Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
s = workloads.cfg4_setup()
models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
spec = workloads.replay_spec(nt, n_steps=ns, seed=2605)
a = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], s["cfg"])


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return min(ms)


out = {}
d1 = torch.empty(nt * SUMMARY_DT.itemsize, dtype=torch.uint8, device="cuda")
ms = timed(lambda: replay_device(ctx, models, *a, spec, d1.data_ptr()))
out["thread"] = nt * ns / (ms * 1e-3)
ctx.set_replay_layout("warp")
d2 = torch.empty_like(d1)
ms = timed(lambda: replay_device(ctx, models, *a, spec, d2.data_ptr()), 1)
out["warp"] = nt * ns / (ms * 1e-3)
ctx.set_replay_layout("thread")
consts = workloads.plant_constants(ctx, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                   s["batches"])
tr, sig = workloads.synthetic_traces(spec, len(models), *consts)
d_tr = torch.from_numpy(tr.view(np.uint8)).cuda()
d_sig = torch.from_numpy(sig.view(np.uint8)).cuda()
d3 = torch.empty_like(d1)
b = TraceBatch(n_traces=nt, first_step=0, n_steps=ns, n_log_traces=0, interval_s=0.5,
               traces=d_tr.data_ptr(), signal=d_sig.data_ptr(), n_signal=len(sig),
               summaries=d3.data_ptr())
ms = timed(lambda: replay_traces_device(ctx, models, *a, b))
out["traces"] = nt * ns / (ms * 1e-3)
import hashlib  # noqa: E402
print("summary sha", hashlib.sha256(d1.cpu().numpy().tobytes()).hexdigest()[:16])
print({k: f"{v:.4g}" for k, v in out.items()},
      "warp==thread", bool(torch.equal(d1, d2)), "traces==thread", bool(torch.equal(d1, d3)))
