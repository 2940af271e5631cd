"""A/B of the step variants (sort chunk x cross-rank vs merge rounds) on the cfg2 step:
device ms/step of plan.run (graph), and selections identical across variants."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21427_b200 import workloads  # noqa: E402
from paper_2605_21427_b200.abi import QUERY_DT  # noqa: E402
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, Grid, Plan  # noqa: E402


def run(chunk, merge, which="cfg2", steps=50):
    os.environ["PALS_SORT_CHUNK"] = str(chunk)
    os.environ["PALS_MERGE"] = str(merge)
    ctx = Context(0)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    c = workloads.cfg2(10_000) if which == "cfg2" else workloads.cfg3_extended()
    plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
    th, _, _ = plan.scores()
    if which == "cfg2":
        q = workloads.gen_queries(10_000, c["seed"], float(th.max()), "qos")
    else:
        q = workloads.gen_queries(10_000, 5, float(th.max()), "mixed", budget=(900.0, 1900.0))
    dq = torch.from_numpy(np.ascontiguousarray(q, QUERY_DT).view(np.uint8)).cuda()
    di = torch.empty(len(q), dtype=torch.int32, device="cuda")
    dr = torch.empty(len(q), dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(st):
        for _ in range(5):
            plan.run(dq.data_ptr(), len(q), di.data_ptr(), dr.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            plan.run(dq.data_ptr(), len(q), di.data_ptr(), dr.data_ptr())
        e1.record(st)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, di.cpu().numpy().copy()


if __name__ == "__main__":
    out = {}
    for which in ("cfg2", "cfg3x"):
        base = None
        for rep in range(2):
            for chunk in (1024, 2048, 4096):
                for merge in (0, 1):
                    ms, idx = run(chunk, merge, which, steps=50 if which == "cfg2" else 10)
                    if base is None:
                        base = idx
                    out[f"{which} chunk{chunk} merge{merge} rep{rep}"] = {
                        "ms": ms, "same": bool(np.array_equal(idx, base))}
                    print(which, chunk, "merge", merge, f"{ms:.4f} ms", np.array_equal(idx, base),
                          flush=True)
    json.dump(out, open(os.environ.get("OUT", "gpurun_out/ab_prep.json"), "w"), indent=1)
