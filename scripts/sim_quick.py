"""Quick GPU check of the queue-plant leg alone: python scripts/sim_quick.py [seeds [bench flags]]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_21427_b200.wattserve import Context  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sys.argv = ["bench.py", "--sim-seeds", str(seeds)] + sys.argv[2:]
args = bench.parse()
d = bench.Dist()
ctx = Context(0)
r = bench.bench_sim(args, d, ctx)
r = r[0] if isinstance(r, tuple) else r
print(json.dumps(r, default=lambda o: o.tolist() if hasattr(o, "tolist") else str(o)))
