"""Find traces where the thread and warp layouts disagree and check them against the C
oracle: python scripts/replay_check.py [n_traces] [n_steps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402
from paper_2605_21427_b200 import workloads  # noqa: E402
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, replay  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 3600
ctx = Context(0)
s = workloads.cfg4_setup()
models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
a = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], s["cfg"])
spec = workloads.replay_spec(nt, n_steps=ns, seed=2605)
th, _ = replay(ctx, models, *a, spec)
ctx.set_replay_layout("warp")
wa, _ = replay(ctx, models, *a, spec)
ctx.set_replay_layout("thread")
bad = np.flatnonzero(th != wa)
print("mismatching traces:", len(bad), bad[:10])
orc = Oracle()
for i in list(bad[:3]) + [0, 1]:
    sp = workloads.replay_spec(1, n_steps=ns, seed=2605, first=int(i))
    o, _ = orc.replay(*a, sp)
    print(i, "thread==oracle", bool(th[i] == o[0]), "warp==oracle", bool(wa[i] == o[0]),
          "obj", int(o[0]["objective"]), "model", int(o[0]["model"]))
