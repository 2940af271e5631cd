"""Run one bench leg alone on GPU 0 (for ncu captures at the bench's sizes):
  python scripts/leg.py alloc|frontier|sim|forest"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21427_b200.wattserve import Context  # noqa: E402

leg = sys.argv[1]
sys.argv = ["bench.py", "--steps", "2", "--warmup", "1"]
args = bench.parse()
dist = bench.Dist()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = Context(0)
ctx.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
l2_flush = flush.zero_
if leg == "alloc":
    out = bench.bench_allocations(args, dist, ctx, stream, l2_flush)
elif leg == "frontier":
    out = bench.bench_frontiers(args, dist, ctx, stream, l2_flush)
elif leg == "sim":
    ctx.set_sim_streaming(False)  # under ncu the launch is serialised with the later uploads
    out = bench.bench_sim(args, dist, ctx)
    out = {k: v for k, v in out.items() if not k.startswith("_")}
elif leg == "forest":
    out, _ = bench.bench_forest(args, dist, ctx, stream, l2_flush)
    out.pop("_kept", None)
else:
    raise SystemExit("unknown leg " + leg)
print(json.dumps(out)[:2000])
