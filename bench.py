#!/usr/bin/env python
"""bench.py — config evals/s (batched select_config) + controller decisions/s
(batched control_step replay) on B200, beside the reference's CPU path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (`value`): cfg2 of BASELINE.json — llama2-7b-like (+tp8), 64 caps x 256
batches x TP{1,2,4,8} = 65,536 configs, 1e4 QoS throughput targets evaluated and
selected in one pass. A step = evaluate the grid (FP64, bit-exact), build the
rank tables, decide all queries; inputs resident in HBM. Unit: (config, query)
pairs actually scanned per second (queries decided without a scan are not
counted). `decisions` (same line): cfg4 — 1e6 traces x 3600 control intervals
through control_step + the fluid plant, one thread per trace.

Multi-GPU (torchrun): weak scaling — every rank runs its own shard of the same
per-GPU workload (queries/traces offset by rank), no collective on the data
path; per-step device time is max-reduced over ranks and rank 0 prints.
`--impl reference`: the reference's own CPU implementation (oracle/_ref, the
unmodified headers) on all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "config evals/sec + controller decisions/sec at 1/2/4/8 B200 vs CPU reference"
SELECT_WORKLOAD = ("cfg2: llama2-7b-like (+tp8 comm), caps 100+300i/63 x batch 1..256 x "
                   "tp{1,2,4,8} = 65536 configs, 1e4 QoS targets per GPU, eval+rank+select "
                   "per step")
ALLOC_WORKLOAD = ("allocate_budget: 1e6 independent clusters per GPU, 1-8 nodes each over the 8 "
                  "calibrated profiles (6x6 candidates at the deployment, dp 1-3), targets "
                  "U(0.2,1) x unconstrained, budgets floors..1.15 x peak, quantum 25 W, "
                  "selection margin 0.02")
REPLAY_WORKLOAD = ("cfg4: 1e6 fluid-plant traces x 3600 control intervals per GPU, 8 calibrated "
                   "profiles, 6x6 candidates each, QoS/budget-throughput 50/50")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--queries", type=int, default=10_000)
    ap.add_argument("--traces", type=int, default=1_000_000)
    ap.add_argument("--trace-steps", type=int, default=3600)
    ap.add_argument("--replay-steps", type=int, default=None,
                    help="timed replay steps (default: min(steps, 5))")
    ap.add_argument("--predictions", type=int, default=1 << 24,
                    help="points per GPU for the forest-predictor leg")
    ap.add_argument("--clusters", type=int, default=1_000_000,
                    help="allocate_budget problems per GPU for the allocator leg")
    ap.add_argument("--cfg3-queries", type=int, default=1_000_000,
                    help="cfg3 (target, budget) queries per GPU")
    ap.add_argument("--cfg5-traces", type=int, default=10_000_000,
                    help="cfg5 traces in total (split over the GPUs)")
    ap.add_argument("--cfg5-steps", type=int, default=2, help="timed cfg5 replays")
    ap.add_argument("--sim-seeds", type=int, default=256,
                    help="seeds per GPU of the 3-scenario x 5-policy queue-plant suite")
    ap.add_argument("--sim-no-stream", action="store_true",
                    help="queue-plant uploads before the launch (for ncu launch lists)")
    ap.add_argument("--sim-steps", type=int, default=2, help="timed queue-plant runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time per reference sample")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers --
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = "nccl"

    def init(self, backend):
        # PALS_BENCH_BACKEND=gloo lets several ranks share one GPU (CI of the N>1 path)
        self.backend = os.environ.get("PALS_BENCH_BACKEND", backend)
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group(self.backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        return self._reduce(x, "max")

    def sum(self, x: float) -> float:
        return self._reduce(x, "sum")

    def _reduce(self, x, op):
        if not self.pg:
            return x
        import torch
        dev = "cuda" if (torch.cuda.is_available() and self.backend == "nccl") else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX if op == "max" else self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks_json():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_metric(kernel: str, key: str):
    """One metric of a kernel from the committed ncu --set full summary (None if absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(kernel, {}).get(key)
    except Exception:
        return None


def ncu_traffic(kernel: str):
    """Per-launch DRAM bytes of a kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# --------------------------------------------------------------- our arm --
def run_ours(args, dist: Dist):
    import torch

    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.abi import QUERY_DT, SUMMARY_DT
    from paper_2605_21427_b200.wattserve import (AnalyticModel, Context, Grid, Plan,
                                                 measure_peaks, replay, replay_device)

    ndev = torch.cuda.device_count()
    if dist.world > ndev and os.environ.get("PALS_BENCH_BACKEND") != "gloo":
        sys.exit(f"bench.py: {dist.world} ranks but {ndev} visible GPUs (one rank per GPU; "
                 "PALS_BENCH_BACKEND=gloo lets CI ranks share one)")
    dev = dist.local % max(1, ndev)  # ranks share a GPU only under the gloo CI override
    torch.cuda.set_device(dev)
    dist.init("nccl")
    # a real (non-legacy-default) stream shared by torch and libpals_gpu, so the CUDA
    # events below bracket exactly the kernels the library launches
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = Context(dev)
    ctx.set_stream(stream.cuda_stream)
    int_peak, fp64_peak = measure_peaks(ctx)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def l2_flush():
        flush.zero_()

    # ---------------- cfg2 select ----------------
    cfg = workloads.cfg2(args.queries)
    plan = Plan(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, cfg["points"]),
                cfg["coeffs"])
    n_cfg = len(cfg["points"])
    th, _, _ = plan.scores()
    tref = float(th.max())
    nq = args.queries
    q = workloads.gen_queries(nq, cfg["seed"], tref, "qos", first=dist.rank * nq)
    d_q = torch.from_numpy(q.view(np.uint8).copy()).cuda()
    d_idx = torch.empty(nq, dtype=torch.int32, device="cuda")
    d_rs = torch.empty(nq, dtype=torch.uint8, device="cuda")

    def select_step():
        # one pass: evaluate the grid, rank it, decide every query (a cached CUDA graph
        # of the 9 kernels; the scan kernel is bracketed by event-record nodes)
        plan.run(d_q.data_ptr(), nq, d_idx.data_ptr(), d_rs.data_ptr())

    plan.time_scan(True)
    for _ in range(args.warmup):
        l2_flush()
        select_step()
    torch.cuda.synchronize()
    counts = plan.stats()
    scanned_q = int(counts[0] + counts[1] + counts[2])
    pairs_step = scanned_q * n_cfg
    int_ops_step = (2 * counts[0] + 4 * counts[1] + 2 * counts[2]) * n_cfg
    clocks = Clocks(dev)
    clocks.start()
    launches0 = ctx.launches
    scan_ms = []
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2))
          for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        l2_flush()
        ev[k][0].record(stream)
        select_step()
        ev[k][1].record(stream)
        scan_ms.append(plan.scan_ms())  # syncs on the scan's end event (outside the step)
    torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    exact_q = int(plan.stats()[5])
    # diagnostic split (not the headline): the same step as separate launches
    plan.time_scan(False)
    prep_ms, split_ms = [], []
    for _ in range(3):
        l2_flush()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        plan.prepare()
        e[1].record(stream)
        plan.select_device(d_q.data_ptr(), nq, d_idx.data_ptr(), d_rs.data_ptr())
        e[2].record(stream)
        torch.cuda.synchronize()
        prep_ms.append(e[0].elapsed_time(e[1]))
        split_ms.append(e[0].elapsed_time(e[2]))
    gather = None
    if dist.world > 1:
        # the only cross-GPU traffic: one gather of (index, reason) per query to rank 0
        from paper_2605_21427_b200.shard import gather_to_rank0
        packed = (d_idx.to(torch.int64) << 8) | d_rs.to(torch.int64)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        if dist.backend != "nccl":
            packed = packed.cpu()
        out_all = gather_to_rank0(packed, nq * dist.world, dist.rank, dist.world)
        g1.record(stream)
        torch.cuda.synchronize()
        gather = {"bytes": nq * dist.world * 8, "ms": g0.elapsed_time(g1), "backend": dist.backend,
                  "rows": None if out_all is None else int(out_all.shape[0])}
    t_rank = float(np.sum(step_ms))
    t_max = dist.max(t_rank)
    pairs_total = dist.sum(float(pairs_step)) * args.steps
    value = pairs_total / (t_max * 1e-3)

    # e2e through the public host-buffer API (pinned host queries -> H2D -> eval+rank+select
    # -> D2H index/reason)
    h_q = torch.empty(nq * QUERY_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    h_qn = h_q.numpy().view(QUERY_DT)
    h_qn[:] = q
    h_idx = torch.empty(nq, dtype=torch.int32, pin_memory=True).numpy()
    h_rs = torch.empty(nq, dtype=torch.uint8, pin_memory=True).numpy()
    from paper_2605_21427_b200.abi import ptr
    lib = ctx.lib

    def e2e_step():
        rc = lib.pals_select(plan.h, ptr(h_qn), nq, ptr(h_idx), ptr(h_rs))
        assert rc == 0, lib.pals_last_error()

    for _ in range(args.warmup):
        e2e_step()
    e2e_ms = []
    for _ in range(args.steps):
        l2_flush()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_max = dist.max(float(np.sum(e2e_ms)))
    e2e_value = pairs_total / (e2e_max * 1e-3)

    scan_avg = float(np.mean(scan_ms))
    roof_counts = (counts, n_cfg, scan_avg)
    time_to_decide = decide_leg(args, dist, plan, d_q, nq, h_qn, stream, l2_flush, None, n_cfg)
    time_to_decide["scan_path"] = {"ms_per_step": t_max / args.steps,
                                   "queries_per_s": dist.sum(float(nq)) * args.steps / (t_max * 1e-3),
                                   "e2e_queries_per_s": dist.sum(float(nq)) * args.steps /
                                   (e2e_max * 1e-3)}
    scan_extra = {"scan_share_of_step": scan_avg / float(np.mean(step_ms)),
                  "step_breakdown_ms": {"graph_step": float(np.mean(step_ms)),
                                        "scan_kernel": scan_avg,
                                        "ungraphed_step": float(np.mean(split_ms)),
                                        "ungraphed_prepare(eval+rank)": float(np.mean(prep_ms))},
                  "chain_peak_secondary": {
                      "value": int_peak / 1e12, "unit": "Tops/s (2 per pair)",
                      "frac": (int_ops_step / (scan_avg * 1e-3)) / int_peak,
                      "source": "pals_measure_peaks: dependent chains of the class-A mix "
                                "(measured; includes the chain's own index arithmetic)"}}

    # ---------------- cfg4 replay ----------------
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    nt = args.traces
    spec = workloads.replay_spec(nt, n_steps=args.trace_steps, seed=2605, first=dist.rank * nt)
    d_sum = torch.empty(nt * SUMMARY_DT.itemsize, dtype=torch.uint8, device="cuda")
    rsteps = args.replay_steps or min(args.steps, 5)
    for _ in range(max(1, min(args.warmup, 2))):
        replay_device(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                      s["batches"], s["cfg"], spec, d_sum.data_ptr())
    torch.cuda.synchronize()
    rev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(rsteps)]
    dist.barrier()
    rl0 = ctx.launches
    for k in range(rsteps):
        l2_flush()
        rev[k][0].record(stream)
        replay_device(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                      s["batches"], s["cfg"], spec, d_sum.data_ptr())
        rev[k][1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    rlaunches = ctx.launches - rl0
    r_ms = [a.elapsed_time(b) for a, b in rev]
    clk = clocks.stop()
    roof = dict(scan_roofline(*roof_counts, clk), **scan_extra)

    r_max = dist.max(float(np.sum(r_ms)))
    dec_total = dist.sum(float(nt) * args.trace_steps) * rsteps
    dec_value = dec_total / (r_max * 1e-3)
    # e2e: host summaries (D2H 48 B/trace into pinned memory); trace inputs are generated
    # from (seed, index) on the device, so nothing crosses H2D
    h_sum = torch.empty(nt * SUMMARY_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    h_sumn = h_sum.numpy().view(SUMMARY_DT)
    replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
           s["cfg"], spec, summaries=h_sumn)  # warm-up
    re2e = []
    for _ in range(min(rsteps, 3)):
        l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
               s["cfg"], spec, summaries=h_sumn)
        b.record(stream)
        b.synchronize()
        re2e.append(a.elapsed_time(b))
    re2e_max = dist.max(float(np.mean(re2e)))
    dec_e2e = dist.sum(float(nt) * args.trace_steps) / (re2e_max * 1e-3)
    # the same cfg4 traces through the warp-per-trace layout, and both layouts on the
    # demand-response scenario's 1,464-candidate grid (SURVEY §8(d) cfg4 variants)
    layouts = replay_layouts(args, dist, ctx, stream, l2_flush, models, s, spec, dec_value)
    args._synthetic_dec_value = dec_value
    traces_leg = bench_traces(args, dist, ctx, stream, l2_flush, models, s, spec, d_sum)
    dec_roof = issue_roofline("k_replay", dec_value / dist.world, "decisions", clk,
                              "instruction issue: one dependent chain of FP64 PID arithmetic, "
                              "table lookups and the plant per trace and step; the FP64 pipe "
                              "runs at ~20 % of its peak (ncu), HBM is idle")

    # ---------------- K2: PredictorBundle::predict throughput ----------------
    predictions, bundle = bench_forest(args, dist, ctx, stream, l2_flush)

    # ---------------- allocate_budget over many clusters ----------------
    allocations = bench_allocations(args, dist, ctx, stream, l2_flush)
    frontiers = bench_frontiers(args, dist, ctx, stream, l2_flush)
    cfg3, c3, tref3, gpu_cfg3 = bench_cfg3(args, dist, ctx, stream, l2_flush, int_peak, clk)
    cfg5 = bench_cfg5(args, dist, ctx, stream, l2_flush) if args.cfg5_traces > 0 else None
    scen = bench_sim(args, dist, ctx) if args.sim_seeds > 0 else None

    # ---------------- cfg1: single-call latency (the drop-in's synchronous API) ----------------
    from paper_2605_21427_b200.abi import CtrlState, Point, Telemetry
    from paper_2605_21427_b200.wattserve import control_step, make_targets, select_config
    c1 = workloads.cfg1()
    m1 = AnalyticModel(ctx, c1["profile"], c1["gpu"])
    th1, _, _ = Plan(m1, Grid(ctx, c1["points"]), c1["coeffs"]).scores()
    tgt = make_targets(0.6 * float(th1.max()), 1600.0)
    for _ in range(20):
        select_config(c1["points"], tgt, m1, c1["coeffs"], 1.0, 0.05, 0.02)
    t0 = time.perf_counter()
    for _ in range(200):
        select_config(c1["points"], tgt, m1, c1["coeffs"], 1.0, 0.05, 0.02)
    sel_us = (time.perf_counter() - t0) / 200 * 1e6
    st = CtrlState()
    st.bias = 1.0
    st.current = Point(*c1["points"][-1].tolist())
    ccfg = workloads.cfg4_setup()["cfg"]
    t0 = time.perf_counter()
    for k in range(200):
        _, st = control_step(Telemetry(0.5 * k, 0.55 * float(th1.max())), 0.5 * k, tgt,
                             c1["points"], m1, c1["coeffs"], st, ccfg)
    step_us = (time.perf_counter() - t0) / 200 * 1e6
    latency = {"workload": "cfg1: llama2-7b-like, 6 caps x 6 batches (36 candidates), target 0.6 x "
                           "unconstrained, static 1600 W budget",
               "python_ctypes": {"select_config_us": sel_us, "control_step_us": step_us},
               "note": "one synchronous call: the candidate set is validated, uploaded, scored "
                       "and ranked once and cached; per call the request is posted in mapped "
                       "pinned memory to the resident one-warp server kernel (k_one_server), "
                       "which answers from the set's tables in shared memory; no kernel launch "
                       "per call (launch_per_call_*: pals_ctx_set_one_server(0)); wall clock"}
    cpp = os.path.join(ROOT, "tests", "cpp", "test_adapter")
    if os.path.exists(cpp) and dist.rank == 0:
        try:
            r = subprocess.run([cpp, ROOT, "--latency"], capture_output=True, text=True,
                               timeout=300)
            latency["cpp_drop_in"] = json.loads(r.stdout.strip().splitlines()[-1])
            latency["select_config_us"] = latency["cpp_drop_in"]["select_config_us"]
            latency["control_step_us"] = latency["cpp_drop_in"]["control_step_us"]
        except Exception as e:  # the binary needs the reference headers at build time
            latency["cpp_drop_in"] = {"error": str(e)[:200]}

    out = {
        "metric": METRIC, "value": value, "unit": "config evals/s",
        "n_gpus": dist.world, "gpus_requested": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": select_config_dict(args, dist.world, n_cfg),
        "select_stats": {"scanned_queries_per_gpu": scanned_q, "exact_fold_queries": exact_q},
        "e2e": {"value": e2e_value, "unit": "config evals/s",
                "h2d_bytes_per_step": nq * QUERY_DT.itemsize,
                "d2h_bytes_per_step": nq * 5,
                "api": "pals_select (C ABI, pinned host buffers: one graph, query upload overlapped with eval+rank, decisions stored to the mapped host buffers by the finalize kernel)"},
        "roofline": roof,
        "time_to_decide": time_to_decide,
        "gpu_launches": int(launches),
        "gather": gather,
        "clocks": clk,
        "decisions": {
            "metric": "controller decisions/s", "value": dec_value, "unit": "decisions/s",
            "ms_per_step": r_max / rsteps, "steps": rsteps, "workload": REPLAY_WORKLOAD,
            "traces_per_gpu": nt, "trace_steps": args.trace_steps,
            "e2e": {"value": dec_e2e, "unit": "decisions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": nt * SUMMARY_DT.itemsize,
                    "api": "pals_replay (C ABI, host summaries)"},
            "roofline": dec_roof, "gpu_launches": int(rlaunches), "layouts": layouts,
            "caller_traces": traces_leg},
        "predictions": predictions,
        "allocations": allocations,
        "frontiers": frontiers,
        "cfg3": cfg3,
        "cfg5": cfg5,
        "scenarios": scen,
        "latency": latency,
        "peaks": {"int_ops_per_s": int_peak, "fp64_flops_per_s": fp64_peak,
                  "hbm_gbs_measured": measured_peaks_json().get("hbm_gbs")},
    }
    forest_kept = predictions.pop("_kept", {})
    cfg5_summ = cfg5.pop("_summaries", None) if cfg5 else None
    sim_nres = scen.pop("_node_results", None) if scen else None
    sim_res = scen.pop("_results", None) if scen else None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        # the reference legs time the unmodified code on the same inputs; their results are
        # kept and compared with the GPU results of the same queries / traces / scenarios
        r2, r4, r3, rs = {}, {}, {}, {}
        out["cpu_baseline"] = cpu_select(args, cfg, tref, args.cpu_seconds, results=r2)
        out["decisions"]["cpu_baseline"] = cpu_replay(args, args.cpu_seconds, results=r4)
        out["predictions"]["cpu_baseline"] = cpu_predict(args, bundle, args.cpu_seconds)
        out["allocations"]["cpu_baseline"] = cpu_allocate(args, args.cpu_seconds)
        out["frontiers"]["cpu_baseline"] = cpu_frontier(args.cpu_seconds)
        out["cfg3"]["cpu_baseline"] = cpu_cfg3(args, c3, tref3, args.cpu_seconds, results=r3)
        if cfg5 is not None:  # same per-trace work as cfg4: the cfg4 reference sample
            out["cfg5"]["cpu_baseline"] = dict(out["decisions"]["cpu_baseline"])
        if scen is not None:
            out["scenarios"]["cpu_baseline"] = cpu_sim(args, args.cpu_seconds, results=rs)
        out["latency"]["cpu_reference_select_config_us"] = cpu_latency(c1, float(th1.max()))
        for leg, cb in ((out["time_to_decide"], out["cpu_baseline"]),
                        (out["cfg3"]["time_to_decide"], out["cfg3"]["cpu_baseline"])):
            if cb.get("value"):
                n_c = out["config"]["configs"]
                leg["reference_queries_per_s"] = cb["value"] / n_c
                leg["e2e_speedup_vs_reference"] = leg["e2e"]["queries_per_s"] / (cb["value"] / n_c)
        out["parity"] = bench_parity(args, r2, (h_idx, h_rs), r3, gpu_cfg3, r4, h_sumn,
                                     cfg5_summ, rs, sim_nres, sim_res)
        out["parity"].update(forest_parity(bundle, forest_kept))
    if dist.rank == 0:
        print(json.dumps(out), flush=True)
    dist.close()


def bench_parity(args, r2, g2, r3, g3, r4, g4, g5, rs, g_nres, g_res):
    """Bench-scale parity: every decision / trace summary / scenario result the reference
    legs computed on this box, compared with the GPU's for the same inputs (the public
    host-buffer API's outputs for cfg2 / cfg3 / cfg4). Plus one extra reference shard at the
    far end of cfg5's 1e7 traces (global trace offsets)."""
    par = {}
    if r2.get("index") is not None:
        n = len(r2["index"])
        p = parity_of(g2[0][:n], r2["index"])
        p["mismatches"] += int((g2[1][:n] != r2["reason"]).sum())
        p["what"] = "cfg2 select_config decisions (index and reason) of the reference sample"
        par["cfg2"] = p
    if r3.get("index") is not None:
        n = len(r3["index"])
        p = parity_of(g3[0][:n], r3["index"])
        p["mismatches"] += int((g3[1][:n] != r3["reason"]).sum())
        p["what"] = "cfg3 decisions, the prefix of the 1e6 queries the reference decided"
        par["cfg3"] = p
    if r4.get("summaries") is not None:
        par["cfg4"] = dict(parity_of(g4, r4["summaries"]),
                           what="cfg4 per-trace summaries (control-step digest, final bias and "
                                "point, energy, tokens, applied count)")
    if g5 is not None and r4.get("summaries") is not None:
        # cfg5 trace i is cfg4 trace i (same generator and seed): the head of cfg5 against
        # the cfg4 sample, the tail against one more reference shard
        from oracle.oracle import Reference
        from paper_2605_21427_b200 import workloads
        s = workloads.cfg4_setup()
        n_tail = min(20_000, len(g5))
        spec = workloads.replay_spec(n_tail, n_steps=args.trace_steps, seed=2605,
                                     first=len(g5) - n_tail)
        _, tail = Reference().bench_replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                           s["batches"], s["cfg"], spec, os.cpu_count() or 1)
        head = parity_of(g5, r4["summaries"])
        tl = parity_of(g5[len(g5) - n_tail:], tail)
        par["cfg5"] = {"checked": head["checked"] + tl["checked"],
                       "mismatches": head["mismatches"] + tl["mismatches"],
                       "against": head["against"],
                       "what": f"cfg5 per-trace summaries: the first {head['checked']} and the "
                               f"last {tl['checked']} of {len(g5)} traces"}
    if rs.get("results") is not None and g_nres is not None:
        # the reference's MetricsSummary / RunSummary fields (final_idx and
        # n_budget_changes are GPU-side bookkeeping the harness does not fill)
        nf = ["tokens_per_joule", "qos_violation_rate", "power_tracking_mae_w", "total_tokens",
              "total_energy_j", "mean_throughput_tps", "throughput_target_tps", "final_bias",
              "arrival_stream_hash", "n_requests", "n_completed", "n_applied"]
        rf = ["tokens_per_joule", "qos_violation_rate", "power_tracking_mae_w", "total_tokens",
              "total_energy_j", "mean_throughput_tps", "cluster_tracking_mae_w",
              "sim_total_energy_j", "n_intervals"]
        from numpy.lib.recfunctions import repack_fields
        nn, ns = len(rs["node_results"]), len(rs["results"])
        pn = parity_of(repack_fields(g_nres[:nn][nf]), repack_fields(rs["node_results"][nf]))
        pr = parity_of(repack_fields(g_res[:ns][rf]), repack_fields(rs["results"][rf]))
        par["scenarios"] = {"checked": pr["checked"], "mismatches": pr["mismatches"] +
                            pn["mismatches"], "against": pr["against"],
                            "what": f"run_scenario RunSummary of {pr['checked']} scenarios and "
                                    f"{pn['checked']} node summaries"}
    return par


def forest_parity(bundle, kept):
    """The forest leg's predictions (cell table and literal walk) against the unmodified
    PredictorBundle::predict on the same points, bit for bit (T and P)."""
    from oracle.oracle import Reference, ref_bundle_predict
    path = os.path.join(tempfile.gettempdir(), "pals_bench_bundle_parity.json")
    bundle.to_json(path)
    ref = Reference()
    out = {}
    for direct, (pts, T, P) in kept.items():
        rT, rP, _ = ref_bundle_predict(ref, path, "mixtral-8x7b-like", pts)
        bad = (T.view(np.uint64) != rT.view(np.uint64)) | (P.view(np.uint64) != rP.view(np.uint64))
        out["forest_direct_walk" if direct else "forest_cells"] = {
            "checked": int(len(pts)), "mismatches": int(bad.sum()),
            "against": "oracle/_ref (the unmodified reference headers)",
            "what": "PredictorBundle::predict T and P bits, default 100-tree bundle"}
    return out


def replay_layouts(args, dist, ctx, stream, l2_flush, models, s, spec, thread_value):
    """decisions/s of the cfg4 replay per kernel layout (thread / warp per trace) and on
    the 1,464-candidate DR grid; same traces, identical results (tests/)."""
    import torch
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.abi import SUMMARY_DT
    from paper_2605_21427_b200.wattserve import replay_device

    def timed(caps, batches, sp, layout, reps):
        ctx.set_replay_layout(layout)
        d = torch.empty(sp.n_traces * SUMMARY_DT.itemsize, dtype=torch.uint8, device="cuda")
        run = lambda: replay_device(ctx, models, s["profiles"], s["gpu"], s["coeffs"],  # noqa
                                    caps, batches, s["cfg"], sp, d.data_ptr())
        run()
        torch.cuda.synchronize()
        dist.barrier()
        ms = 0.0
        for _ in range(reps):
            l2_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run()
            b.record(stream)
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        ctx.set_replay_layout("thread")
        t = dist.max(ms)
        return dist.sum(float(sp.n_traces) * sp.n_steps) * reps / (t * 1e-3)

    out = {"cfg4_thread_per_trace": thread_value,
           "cfg4_warp_per_trace": timed(s["caps"], s["batches"], spec, "warp", 2)}
    caps, batches = workloads.dr_candidates()
    nt = max(1, args.traces // 4)
    dspec = workloads.replay_spec(nt, n_steps=args.trace_steps, seed=2605,
                                  first=dist.rank * nt)
    out["dr_grid_workload"] = (f"{nt} traces per GPU x {args.trace_steps} steps on the "
                               f"demand-response grid: 61 caps x 24 batches = 1,464 candidates")
    out["dr_thread_per_trace"] = timed(caps, batches, dspec, "thread", 2)
    out["dr_warp_per_trace"] = timed(caps, batches, dspec, "warp", 1)
    out["unit"] = "decisions/s"
    return out


def bench_traces(args, dist, ctx, stream, l2_flush, models, s, spec, d_synth):
    """cfg4 through the caller-trace boundary (pals_replay_traces): the same 1e6 traces,
    written out as caller budget / load signals (446 MB of (t_s, value) rows + 64 B per
    trace), device-resident for `value`; `e2e` from pinned host buffers through the host
    call, which also returns every final ControllerState and plant state. Parity: every
    trace summary equals the synthetic path's (d_synth) bit for bit."""
    import torch
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.abi import (PLANT_DT, SIGNAL_DT, STATE_DT, SUMMARY_DT, TRACE_DT,
                                           TraceBatch)
    from paper_2605_21427_b200.wattserve import replay_traces_device
    consts = workloads.plant_constants(ctx, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                       s["batches"])
    tr, sig = workloads.synthetic_traces(spec, len(models), *consts)
    nt = len(tr)
    d_tr = torch.from_numpy(tr.view(np.uint8)).cuda()
    d_sig = torch.from_numpy(sig.view(np.uint8)).cuda()
    d_sum = torch.empty(nt * SUMMARY_DT.itemsize, dtype=torch.uint8, device="cuda")
    d_fin = torch.empty(nt * STATE_DT.itemsize, dtype=torch.uint8, device="cuda")
    d_finp = torch.empty(nt * PLANT_DT.itemsize, dtype=torch.uint8, device="cuda")
    b = TraceBatch(n_traces=nt, first_step=0, n_steps=spec.n_steps, n_log_traces=0,
                   interval_s=spec.interval_s, traces=d_tr.data_ptr(), signal=d_sig.data_ptr(),
                   n_signal=len(sig), init=None, init_plant=None, summaries=d_sum.data_ptr(),
                   final_state=d_fin.data_ptr(), final_plant=d_finp.data_ptr(), logs=None,
                   details=None)
    run = lambda: replay_traces_device(ctx, models, s["profiles"], s["gpu"], s["coeffs"],  # noqa
                                       s["caps"], s["batches"], s["cfg"], b)
    run()
    torch.cuda.synchronize()
    reps = max(1, min(args.steps, 3))
    dist.barrier()
    ms = []
    for _ in range(reps):
        l2_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = dist.max(float(np.sum(ms)))
    value = dist.sum(float(nt) * spec.n_steps) * reps / (t * 1e-3)
    mism = int((d_sum != d_synth).view(nt, SUMMARY_DT.itemsize).any(1).sum().item())
    # e2e: pinned host traces / signals in, summaries + final states out, host call
    h_tr = torch.empty(tr.nbytes, dtype=torch.uint8, pin_memory=True)
    h_tr.numpy()[:] = tr.view(np.uint8)
    h_sig = torch.empty(sig.nbytes, dtype=torch.uint8, pin_memory=True)
    h_sig.numpy()[:] = sig.view(np.uint8)
    h_sum = torch.empty(nt * SUMMARY_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    h_fin = torch.empty(nt * STATE_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    h_finp = torch.empty(nt * PLANT_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    hb = TraceBatch(n_traces=nt, first_step=0, n_steps=spec.n_steps, n_log_traces=0,
                    interval_s=spec.interval_s, traces=h_tr.data_ptr(), signal=h_sig.data_ptr(),
                    n_signal=len(sig), init=None, init_plant=None, summaries=h_sum.data_ptr(),
                    final_state=h_fin.data_ptr(), final_plant=h_finp.data_ptr(), logs=None,
                    details=None)
    import ctypes as C
    from paper_2605_21427_b200.wattserve import _replay_common
    n_models, hs, profs, caps, batches = _replay_common(models, s["profiles"], s["caps"],
                                                        s["batches"])
    lib = ctx.lib

    def e2e():
        rc = lib.pals_replay_traces(ctx.h, n_models, hs, profs, C.byref(s["gpu"]),
                                    C.byref(s["coeffs"]), caps.ctypes.data, len(caps),
                                    batches.ctypes.data, len(batches), C.byref(s["cfg"]),
                                    C.byref(hb))
        assert rc == 0, lib.pals_last_error()

    e2e()
    e2e_ms = []
    for _ in range(reps):
        l2_flush()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e()
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    te = dist.max(float(np.mean(e2e_ms)))
    e2e_value = dist.sum(float(nt) * spec.n_steps) / (te * 1e-3)
    mism_e2e = int((h_sum.cuda() != d_synth).view(nt, SUMMARY_DT.itemsize).any(1).sum().item())
    return {"metric": "controller decisions/s over caller traces (pals_replay_traces)",
            "value": value, "unit": "decisions/s", "ms_per_step": t / reps,
            "workload": f"the cfg4 traces ({nt} per GPU x {spec.n_steps} steps) as caller "
                        f"signals: {len(sig)} (t_s, value) rows, {sig.nbytes + tr.nbytes} B",
            "e2e": {"value": e2e_value, "unit": "decisions/s",
                    "h2d_bytes_per_step": int(tr.nbytes + sig.nbytes),
                    "d2h_bytes_per_step": int(nt * (SUMMARY_DT.itemsize + STATE_DT.itemsize +
                                                    PLANT_DT.itemsize)),
                    "api": "pals_replay_traces (C ABI, pinned host traces in; summaries, "
                           "ControllerStates and plant states out)"},
            "vs_synthetic_path": value / max(1.0, float(args._synthetic_dec_value)),
            "parity": {"checked": nt, "mismatches": mism + mism_e2e,
                       "against": "the synthetic replay of the same traces (k_replay, "
                                  "itself checked against oracle/_ref)"}}


def bench_forest(args, dist, ctx, stream, l2_flush):
    """PredictorBundle::predict (forest.hpp:227-235) over random points, on the bundle at the
    reference's default hyper-parameters (100 trees per forest, depth 14; trained by the
    reference pipeline, data/predictor_default.npz): the exact lattice-cell table (the
    default path) and the literal tree walk, plus the shipped 20-tree bundle."""
    import torch
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.forest import Bundle, make_forest_model
    data = os.path.join(ROOT, "paper_2605_21427_b200", "data")
    bundle = Bundle.load_npz(os.path.join(data, "predictor_default.npz"))
    small = Bundle.load_npz(os.path.join(data, "predictor_small.npz"))
    hbm = measured_peaks_json().get("hbm_gbs", 6552.6)

    def timed(model, npts, direct, reps, keep=True):
        ctx.lib.pals_model_forest_set_direct(model.h, 1 if direct else 0)
        pts = workloads.predict_points(npts, seed=2605 + dist.rank)
        d_pts = torch.from_numpy(pts.view(np.uint8)).cuda()
        d_T = torch.empty(npts, dtype=torch.float64, device="cuda")
        d_P = torch.empty(npts, dtype=torch.float64, device="cuda")

        def step():
            rc = ctx.lib.pals_predict_device(ctx.h, model.h, d_pts.data_ptr(), npts,
                                             d_T.data_ptr(), d_P.data_ptr())
            assert rc == 0, ctx.lib.pals_last_error()

        for _ in range(max(1, args.warmup)):
            step()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(reps)]
        dist.barrier()
        for k in range(reps):
            l2_flush()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        t = dist.max(float(np.sum([a.elapsed_time(b) for a, b in ev])))
        ctx.lib.pals_model_forest_set_direct(model.h, 0)
        if keep:  # the default bundle's predictions, for the parity check
            k = min(npts, 50_000)
            kept[direct] = (pts[:k], d_T[:k].cpu().numpy(), d_P[:k].cpu().numpy())
        return dist.sum(float(npts)) * reps / (t * 1e-3), t / reps

    kept = {}
    mid = "mixtral-8x7b-like"
    fmodel = make_forest_model(ctx, bundle, mid)
    npred = args.predictions
    value, ms = timed(fmodel, npred, False, args.steps)
    n_direct = max(1, npred // 16)
    v_direct, ms_direct = timed(fmodel, n_direct, True, max(1, min(args.steps, 3)))
    smodel = make_forest_model(ctx, small, mid)
    v_small, _ = timed(smodel, npred, False, args.steps, keep=False)
    nodes = int(sum(len(f.feature) for f in (bundle.throughput, bundle.power)))
    depth = bundle.hyperparams["max_depth"]
    pred_bytes = 40.0  # 24 B point in, 16 B T/P out: the cell path's algorithmic traffic
    per_gpu = value / dist.world
    return {
        "metric": "predictor predictions/s (PredictorBundle::predict, T and P)",
        "value": value, "unit": "predictions/s", "ms_per_step": ms, "points_per_gpu": npred,
        "bundle": f"{bundle.throughput.n_trees}+{bundle.power.n_trees} trees, depth {depth}, "
                  f"{nodes} nodes (the reference's default hyper-parameters, trained by its "
                  f"own pipeline); {int(ctx.lib.pals_model_forest_cells(fmodel.h))} exact "
                  "lattice cells",
        "roofline": {"bound": "hbm", "kernel": "k_forest_eval_aos",
                     "achieved": per_gpu * pred_bytes / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": per_gpu * pred_bytes / 1e9 / hbm,
                     "traffic": ncu_traffic("k_forest_eval_aos"),
                     "algorithmic": "40 B per prediction (24 B point in, 16 B T/P out)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "direct_walk": {"value": v_direct, "unit": "predictions/s", "points_per_gpu": n_direct,
                        "ms_per_step": ms_direct,
                        "note": "the literal per-point walk of all 200 trees (forest.hpp:80-85, "
                                "176-180), used when a bundle's lattice exceeds 4M cells",
                        "tree_node_visits_per_s": v_direct * 200 * depth},
        "small_bundle": {"value": v_small, "unit": "predictions/s",
                         "bundle": f"{small.throughput.n_trees}+{small.power.n_trees} trees, "
                                   f"depth {small.hyperparams['max_depth']} (predictor_small)"},
        "_kept": kept,
    }, bundle


def alloc_setup_gpu(ctx):
    """Allocator + per-model scales (unconstrained t_hat, peak p_node at dp 1) from the GPU."""
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.wattserve import Allocator, AnalyticModel, Grid, Plan
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    tm, pm = [], []
    for p, m in zip(s["profiles"], models):
        pts = workloads.grid_points(s["caps"], s["batches"], [p.deploy_tp], [p.deploy_ep], [1])
        th, pn, _ = Plan(m, Grid(ctx, pts), s["coeffs"]).scores()
        tm.append(float(th.max()))
        pm.append(float(pn.max()))
    al = Allocator(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                   max_dp=3, selection_margin=0.02)
    return s, al, tm, pm


def bench_allocations(args, dist, ctx, stream, l2_flush):
    import torch
    from paper_2605_21427_b200 import workloads
    s, al, tm, pm = alloc_setup_gpu(ctx)
    n = args.clusters
    prob = workloads.alloc_problems(n, 2605, tm, pm, s["gpu"], s["coeffs"], first=dist.rank * n)
    nn = int(prob["off"][-1])
    host = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in
            (("off", prob["off"]), ("model", prob["model"]), ("dp", prob["dp"]),
             ("target", prob["target"]), ("budget", prob["budget"]))}
    dev = {k: v.cuda() for k, v in host.items()}
    pin = {k: v.pin_memory() for k, v in host.items()}
    out_d = dict(nb=torch.empty(nn, dtype=torch.float64, device="cuda"),
                 tot=torch.empty(n, dtype=torch.float64, device="cuda"),
                 sat=torch.empty(n, dtype=torch.uint8, device="cuda"),
                 st=torch.empty(n, dtype=torch.int32, device="cuda"))
    out_h = dict(nb=torch.empty(nn, dtype=torch.float64).pin_memory(),
                 tot=torch.empty(n, dtype=torch.float64).pin_memory(),
                 sat=torch.empty(n, dtype=torch.uint8).pin_memory(),
                 st=torch.empty(n, dtype=torch.int32).pin_memory())

    def step():
        al.run_device(25.0, n, nn, dev["off"].data_ptr(), dev["model"].data_ptr(),
                      dev["dp"].data_ptr(), dev["target"].data_ptr(), dev["budget"].data_ptr(),
                      out_d["nb"].data_ptr(), out_d["tot"].data_ptr(), out_d["sat"].data_ptr(),
                      out_d["st"].data_ptr())

    def e2e_step():
        rc = ctx.lib.pals_allocate_budget(
            al.h, 25.0, n, pin["off"].data_ptr(), pin["model"].data_ptr(), pin["dp"].data_ptr(),
            pin["target"].data_ptr(), pin["budget"].data_ptr(), out_h["nb"].data_ptr(),
            out_h["tot"].data_ptr(), out_h["sat"].data_ptr(), out_h["st"].data_ptr())
        assert rc == 0, ctx.lib.pals_last_error()

    for _ in range(args.warmup):
        step()
        e2e_step()
    torch.cuda.synchronize()
    l0 = ctx.lib.pals_ctx_launch_count(ctx.h)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for k in range(args.steps):
        l2_flush()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    launches = ctx.lib.pals_ctx_launch_count(ctx.h) - l0
    t_max = dist.max(float(np.sum([a.elapsed_time(b) for a, b in ev])))
    value = dist.sum(float(n)) * args.steps / (t_max * 1e-3)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_t = dist.max(time.perf_counter() - t0)
    e2e = dist.sum(float(n)) * args.steps / e2e_t
    status = out_h["st"].numpy()
    # algorithmic bytes per cluster: offsets 8 + budget 8 + per node (model 4 + dp 4 +
    # target 8 in, budget 8 out) + total 8 + flag 1 + status 4 out
    nbytes = (8 + 8 + 8 + 1 + 4) * n + 24 * nn
    hbm = measured_peaks_json().get("hbm_gbs", 6552.6)
    ach = nbytes / (t_max * 1e-3 / args.steps) / 1e9
    return {
        "metric": "cluster budget allocations/s (allocate_budget, water-filling)",
        "value": value, "unit": "allocations/s", "ms_per_step": t_max / args.steps,
        "steps": args.steps, "workload": ALLOC_WORKLOAD, "clusters_per_gpu": n,
        "nodes_per_gpu": nn, "ok_fraction": float((status == 0).mean()),
        "e2e": {"value": e2e, "unit": "allocations/s",
                "h2d_bytes_per_step": int(8 * (n + 1) + 16 * nn + 8 * n),
                "d2h_bytes_per_step": int(8 * nn + 13 * n),
                "api": "pals_allocate_budget (C ABI, pinned host buffers)"},
        "roofline": dict(issue_roofline("k_allocate", value / dist.world, "allocations", None,
                                        "instruction issue: the reference's serial greedy "
                                        "loop per cluster (one thread per cluster), FP64 "
                                        "divides in the marginal-rate comparisons"),
                         hbm_bytes_secondary={"algorithmic": "29 B per cluster + 24 B per node",
                                              "achieved_gbs": ach, "peak_gbs": hbm,
                                              "frac": ach / hbm}),
        "gpu_launches": int(launches),
    }


CFG3_WORKLOAD = ("cfg3: mixtral-8x7b-like MoE (+tp8 comm), caps 100+300i/63 x batch 1..256 x "
                 "tp{1,2,4,8} at ep=8 = 65536 configs, 1e6 (target, budget) queries per GPU, "
                 "QoS / budget-throughput 50/50, budget U(600,2000) W, margin 0.02; "
                 "eval+rank+select per step")
CFG5_WORKLOAD = ("cfg5: 1e7 fluid-plant traces in total (8 calibrated profiles: dense and MoE) x "
                 "3600 control intervals, contiguous trace shards per GPU, final per-trace "
                 "summary gather (48 B/trace) to rank 0")


def bench_cfg3(args, dist, ctx, stream, l2_flush, int_peak, clk=None):
    """BASELINE cfg3: the MoE grid with 1e6 mixed (target, budget) queries per GPU."""
    import torch
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.abi import QUERY_DT, ptr
    from paper_2605_21427_b200.wattserve import AnalyticModel, Grid, Plan
    c = workloads.cfg3(args.cfg3_queries)
    plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
    n_cfg = len(c["points"])
    th, _, _ = plan.scores()
    tref = float(th.max())
    nq = args.cfg3_queries
    q = workloads.gen_queries(nq, c["seed"], tref, c["objective"], budget=c["budget"],
                              first=dist.rank * nq)
    d_q = torch.from_numpy(q.view(np.uint8).copy()).cuda()
    d_idx = torch.empty(nq, dtype=torch.int32, device="cuda")
    d_rs = torch.empty(nq, dtype=torch.uint8, device="cuda")
    step = lambda: plan.run(d_q.data_ptr(), nq, d_idx.data_ptr(), d_rs.data_ptr())  # noqa: E731
    plan.time_scan(True)
    for _ in range(args.warmup):
        l2_flush()
        step()
    torch.cuda.synchronize()
    cnt = plan.stats()
    scanned_q = int(cnt[0] + cnt[1] + cnt[2])
    int_ops_step = (2 * cnt[0] + 4 * cnt[1] + 2 * cnt[2]) * n_cfg
    l0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    scan_ms = []
    dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        l2_flush()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
        scan_ms.append(plan.scan_ms())
    torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launches - l0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_max = dist.max(float(np.sum(step_ms)))
    pairs_total = dist.sum(float(scanned_q * n_cfg)) * args.steps
    value = pairs_total / (t_max * 1e-3)
    # e2e: pinned host queries -> pals_select (H2D, eval+rank+select, D2H index/reason)
    h_q = torch.empty(nq * QUERY_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    h_qn = h_q.numpy().view(QUERY_DT)
    h_qn[:] = q
    h_idx = torch.empty(nq, dtype=torch.int32, pin_memory=True).numpy()
    h_rs = torch.empty(nq, dtype=torch.uint8, pin_memory=True).numpy()
    lib = ctx.lib

    def e2e_step():
        rc = lib.pals_select(plan.h, ptr(h_qn), nq, ptr(h_idx), ptr(h_rs))
        assert rc == 0, lib.pals_last_error()

    e2e_step()
    e2e_ms = []
    for _ in range(args.steps):
        l2_flush()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_max = dist.max(float(np.sum(e2e_ms)))
    scan_avg = float(np.mean(scan_ms))
    ttd = decide_leg(args, dist, plan, d_q, nq, h_qn, stream, l2_flush, None, n_cfg)
    ttd["scan_path"] = {"ms_per_step": t_max / args.steps,
                        "e2e_queries_per_s": dist.sum(float(nq)) * args.steps / (e2e_max * 1e-3)}
    # strong scaling: the 1e6 queries in total, contiguous shards over the ranks (at N = 1
    # the same work as the weak leg)
    from paper_2605_21427_b200.shard import shard_range
    s_first, s_n = shard_range(nq, dist.rank, dist.world)
    qs = workloads.gen_queries(max(1, s_n), c["seed"], tref, c["objective"], budget=c["budget"],
                               first=s_first)
    d_qs = torch.from_numpy(qs.view(np.uint8).copy()).cuda()
    steps_s = lambda: plan.run(d_qs.data_ptr(), s_n, d_idx.data_ptr(), d_rs.data_ptr())  # noqa
    steps_s()
    torch.cuda.synchronize()
    cnt_s = plan.stats()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    dist.barrier()
    for k in range(args.steps):
        l2_flush()
        evs[k][0].record(stream)
        steps_s()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    ts = dist.max(float(np.sum([e0.elapsed_time(e1) for e0, e1 in evs])))
    pairs_s = dist.sum(float((cnt_s[0] + cnt_s[1] + cnt_s[2]) * n_cfg)) * args.steps
    strong = {"scaling": "strong", "queries_total": nq, "queries_this_rank": s_n,
              "value": pairs_s / (ts * 1e-3), "unit": "config evals/s",
              "ms_per_step": ts / args.steps,
              "queries_per_s": float(nq) * args.steps / (ts * 1e-3)}
    # the optional EP x DP extension of cfg3: 589,824 configs, 64-bit keys
    cx = workloads.cfg3_extended()
    planx = Plan(AnalyticModel(ctx, cx["profile"], cx["gpu"]), Grid(ctx, cx["points"]),
                 cx["coeffs"])
    thx, _, _ = planx.scores()
    nqx = max(1, min(nq, 10_000))
    qx = workloads.gen_queries(nqx, c["seed"], float(thx.max()), c["objective"],
                               budget=c["budget"], first=dist.rank * nqx)
    d_qx = torch.from_numpy(qx.view(np.uint8).copy()).cuda()
    stepx = lambda: planx.run(d_qx.data_ptr(), nqx, d_idx.data_ptr(), d_rs.data_ptr())  # noqa
    stepx()
    torch.cuda.synchronize()
    cx_cnt = planx.stats()
    evx = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for k in range(args.steps):
        l2_flush()
        evx[k][0].record(stream)
        stepx()
        evx[k][1].record(stream)
    torch.cuda.synchronize()
    tx = dist.max(float(np.sum([e0.elapsed_time(e1) for e0, e1 in evx])))
    pairs_x = dist.sum(float((cx_cnt[0] + cx_cnt[1] + cx_cnt[2]) * len(cx["points"]))) * args.steps
    extended = {"workload": "cfg3 x EP{1,4,8} x DP{1,2,3}: 589,824 configs (64-bit packed keys), "
                            f"{nqx} mixed queries per GPU, eval+rank+select per step",
                "value": pairs_x / (tx * 1e-3), "unit": "config evals/s",
                "ms_per_step": tx / args.steps, "queries_per_gpu": nqx}
    out = {"metric": "config evals/s (cfg3 select_config, MoE grid, mixed QoS/budget queries)",
           "value": value, "unit": "config evals/s", "ms_per_step": t_max / args.steps,
           "steps": args.steps, "workload": CFG3_WORKLOAD, "configs": n_cfg,
           "queries_per_gpu": nq, "scanned_queries_per_gpu": scanned_q,
           "query_classes": {"qos_no_budget": int(cnt[0]), "qos_budget": int(cnt[1]),
                             "budget_only": int(cnt[2]), "no_scan": int(cnt[3]),
                             "exact_fold": int(cnt[5])},
           "e2e": {"value": pairs_total / (e2e_max * 1e-3), "unit": "config evals/s",
                   "h2d_bytes_per_step": nq * QUERY_DT.itemsize, "d2h_bytes_per_step": nq * 5,
                   "api": "pals_select (C ABI, pinned host buffers: one graph, query upload overlapped with eval+rank, decisions stored to the mapped host buffers by the finalize kernel)"},
           "roofline": dict(scan_roofline(cnt, n_cfg, scan_avg, clk),
                            scan_share_of_step=scan_avg / float(np.mean(step_ms))),
           "gpu_launches": int(launches), "extended_grid": extended, "scaling": "weak",
           "strong": strong, "time_to_decide": ttd}
    return out, c, tref, (h_idx, h_rs)


def cpu_cfg3(args, c, tref, seconds, results=None):
    """cfg3 queries through the unmodified select_config + analytic_scorer, all threads."""
    from paper_2605_21427_b200 import workloads
    kind, ref = _reference_backend()
    if kind != "reference":
        return {"value": None, "unit": "config evals/s", "cores": 0, "kind": "port",
                "sample": "reference build absent"}
    threads = os.cpu_count() or 1
    n = len(c["points"])
    q = workloads.gen_queries(4 * threads, c["seed"], tref, c["objective"], budget=c["budget"])
    t, _, _ = ref.bench_select(c["profile"], c["gpu"], c["points"], c["coeffs"], q, threads,
                               want_results=False)
    nq = int(min(args.cfg3_queries, max(threads, len(q) * n / t * seconds / n)))
    q = workloads.gen_queries(nq, c["seed"], tref, c["objective"], budget=c["budget"])
    t, ri, rr = ref.bench_select(c["profile"], c["gpu"], c["points"], c["coeffs"], q, threads,
                                 want_results=results is not None)
    if results is not None:
        results.update(index=ri, reason=rr)
    return {"value": nq * n / t, "unit": "config evals/s", "cores": threads, "kind": "reference",
            "sample": f"first {nq} of the 1e6 cfg3 queries x {n} configs through the unmodified "
                      f"select_config+analytic_scorer, {threads} threads, {t:.1f} s"}


def bench_cfg5(args, dist, ctx, stream, l2_flush):
    """BASELINE cfg5: 1e7 traces in total, strong-scaled over the ranks, plus the one
    result gather (per-trace summaries) to rank 0."""
    import torch
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.abi import SUMMARY_DT
    from paper_2605_21427_b200.shard import gather_to_rank0, shard_range
    from paper_2605_21427_b200.wattserve import AnalyticModel, replay_device
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    n_total = args.cfg5_traces
    first, nt = shard_range(n_total, dist.rank, dist.world)
    spec = workloads.replay_spec(nt, n_steps=args.trace_steps, seed=2605, first=first)
    d_sum = torch.empty((nt, SUMMARY_DT.itemsize), dtype=torch.uint8, device="cuda")
    run = lambda: replay_device(ctx, models, s["profiles"], s["gpu"], s["coeffs"],  # noqa: E731
                                s["caps"], s["batches"], s["cfg"], spec, d_sum.data_ptr())
    run()
    torch.cuda.synchronize()
    steps = args.cfg5_steps
    l0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize()
    for k in range(steps):
        l2_flush()
        ev[k][0].record(stream)
        run()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launches - l0
    t_max = dist.max(float(np.sum([a.elapsed_time(b) for a, b in ev])))
    dec = float(n_total) * args.trace_steps * steps
    # the only cross-GPU traffic: the per-trace summaries to rank 0 (NCCL gather over
    # NVLink; a copy when N = 1)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = (torch.empty((n_total, SUMMARY_DT.itemsize), dtype=torch.uint8, pin_memory=True)
            if dist.rank == 0 else None)
    dist.barrier()
    torch.cuda.synchronize()
    g0.record(stream)
    local = d_sum if dist.backend == "nccl" or dist.world == 1 else d_sum.cpu()
    allsum = gather_to_rank0(local, n_total, dist.rank, dist.world)
    if dist.rank == 0:  # land the gathered summaries in pinned host memory
        host.copy_(allsum, non_blocking=True)
    g1.record(stream)
    torch.cuda.synchronize()
    gather_ms = dist.max(g0.elapsed_time(g1))
    digest = None
    if dist.rank == 0:
        a = host.numpy().reshape(-1).view(SUMMARY_DT)
        # checksum of checksums over all traces (size-independent parity handle)
        h = np.uint64(0xCBF29CE484222325)
        x = np.bitwise_xor.reduce(a["digest"] * np.uint64(0x100000001B3))
        digest = f"{int(h ^ x):016x}"
    return {"metric": "controller decisions/s (cfg5, strong scaling over the GPUs)",
            "value": dec / (t_max * 1e-3), "unit": "decisions/s",
            "ms_per_step": t_max / steps, "steps": steps, "scaling": "strong",
            "workload": CFG5_WORKLOAD, "traces_total": n_total, "traces_this_rank": nt,
            "trace_steps": args.trace_steps,
            "gather": {"bytes": n_total * SUMMARY_DT.itemsize, "ms": gather_ms,
                       "backend": dist.backend if dist.world > 1 else "none (N=1)",
                       "digest_xor": digest},
            "e2e": {"value": dec / steps / ((t_max / steps + gather_ms) * 1e-3),
                    "unit": "decisions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": n_total * SUMMARY_DT.itemsize,
                    "api": "pals_replay_device, then the summary gather to rank 0 and its "
                           "D2H into pinned host memory (the gather+D2H time is added once "
                           "per step)"},
            "gpu_launches": int(launches),
            "_summaries": None if host is None else host.numpy().reshape(-1).view(SUMMARY_DT)}


SIM_WORKLOAD = ("queue-plant run_scenario (sim.hpp) over the 3 bundled scenarios (single_node "
                "900 s x 1 node, multinode_qos 3600 s x 3 nodes, demand_response 3600 s x 3 "
                "nodes on the 1,464-candidate DR grid) x the 5 policies (run_baseline_suite) x "
                "S seeds; predictor = the shipped 20-tree bundle; unit = node control "
                "intervals simulated")


def sim_suite(seeds: int, first_seed: int = 0):
    from paper_2605_21427_b200.abi import POLICIES
    from paper_2605_21427_b200.sim import bundled_scenarios, n_intervals
    base = bundled_scenarios()
    scs = []
    for k in range(seeds):
        for name in sorted(base):
            for pol in POLICIES:
                scs.append(dict(base[name], policy=pol, seed=base[name]["seed"] + first_seed + k))
    units = sum(len(s["nodes"]) * n_intervals(s) for s in scs)
    return scs, units


def sim_predictors(ctx, profiles):
    from paper_2605_21427_b200.forest import Bundle, make_forest_model
    b = Bundle.load_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data",
                                     "predictor_small.npz"))
    return b, {p.name.decode(): make_forest_model(ctx, b, p.name.decode()) for p in profiles}


def bench_sim(args, dist, ctx):
    """Batched run_scenario: whole API call (host arrival streams + budget splits +
    device simulation) and the simulation kernel alone."""
    from paper_2605_21427_b200.profiles import load_bundle
    from paper_2605_21427_b200.sim import last_timing, run_scenarios
    if args.sim_no_stream:
        ctx.set_sim_streaming(False)
    profs, gpu, coeffs = load_bundle()
    _, preds = sim_predictors(ctx, profs)
    scs, units = sim_suite(args.sim_seeds, first_seed=dist.rank * args.sim_seeds)
    # warm-up at the timed size (allocates the context's pinned / device stream buffers)
    run_scenarios(ctx, scs, profs, gpu, coeffs, preds)
    walls, kms, preps = [], [], []
    for _ in range(max(1, args.sim_steps)):
        dist.barrier()
        t0 = time.perf_counter()
        nres, res, _, _ = run_scenarios(ctx, scs, profs, gpu, coeffs, preds)
        walls.append(time.perf_counter() - t0)
        prep, km = last_timing(ctx)
        kms.append(km)
        preps.append(prep)
    wall = dist.max(float(np.mean(walls)))
    km = dist.max(float(np.mean(kms)))
    total = dist.sum(float(units))
    return {"metric": "scenario node-intervals/s (run_scenario queue plant, 5-policy suites)",
            "value": total / (km * 1e-3), "unit": "node-intervals/s",
            "ms_per_step": km, "steps": len(walls), "workload": SIM_WORKLOAD,
            "scenarios_per_gpu": len(scs), "seeds_per_gpu": args.sim_seeds,
            "node_intervals_per_gpu": units,
            "value_basis": "device time of the simulation kernel (k_sim)",
            "roofline": {"bound": "latency", "kernel": "k_sim", "achieved": None, "peak": None,
                         "frac": None, "traffic": ncu_traffic("k_sim"),
                         "note": "each scenario is a sequential chain of 1,800-7,200 intervals "
                                 "with dependent chunk iterations; throughput scales with "
                                 "scenarios in flight (DESIGN.md §5e)",
                         "issue_active_pct_ncu_16_seeds": ncu_metric("k_sim",
                                                                     "issue_active_pct")},
            "e2e": {"value": total / wall, "unit": "node-intervals/s",
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": int(nres.nbytes + res.nbytes),
                    "host_setup_s": float(np.mean(preps)),
                    "api": "pals_run_scenarios (C ABI): host arrival lengths (mt19937_64 + libm, "
                           "all host threads) and budget splits, then k_sim and the arrival "
                           "hashes (k_arrival_hash, side stream); wall clock"},
            "gpu_launches": None, "_node_results": nres, "_results": res}


def cpu_sim(args, seconds, results=None):
    """The unmodified run_scenario + summarize on all host threads over the first seeds of
    the same suite."""
    kind, ref = _reference_backend()
    if kind != "reference":
        return {"value": None, "unit": "node-intervals/s", "cores": 0, "kind": "port",
                "sample": "reference build absent"}
    from paper_2605_21427_b200.profiles import load_bundle
    from paper_2605_21427_b200.forest import Bundle
    profs, gpu, coeffs = load_bundle()
    b = Bundle.load_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data",
                                     "predictor_small.npz"))
    path = os.path.join(tempfile.gettempdir(), "pals_bench_sim_bundle.json")
    b.to_json(path)
    threads = os.cpu_count() or 1
    scs, units = sim_suite(1)
    t = ref.bench_scenarios(scs, profs, gpu, coeffs, path, threads)
    seeds = int(max(1, min(args.sim_seeds, seconds / max(t, 1e-3))))
    if seeds > 1 or results is not None:
        scs, units = sim_suite(seeds)
        out = ref.bench_scenarios(scs, profs, gpu, coeffs, path, threads,
                                  want_results=results is not None)
        if results is not None:  # the sample's node results and RunSummary per scenario
            t, results["node_results"], results["results"] = out
        else:
            t = out
    return {"value": units / t, "unit": "node-intervals/s", "cores": threads,
            "kind": "reference",
            "sample": f"{len(scs)} scenarios ({seeds} seeds x 3 bundled x 5 policies) through "
                      f"the unmodified run_scenario + summarize, {threads} threads, {t:.1f} s"}


FRONTIER_WORKLOAD = ("build_frontier over cfg3x: mixtral-8x7b-like, 64 caps x 256 batches x "
                     "TP{1,2,4,8} x EP{1,4,8} x DP{1,2,3} = 589,824 points scored "
                     "(cluster_throughput, efficiency) and reduced to the Pareto frontier per step")


def bench_frontiers(args, dist, ctx, stream, l2_flush):
    import torch
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.wattserve import AnalyticModel, Grid, Plan
    c = workloads.cfg3_extended()
    n = len(c["points"])
    plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
    d_idx = torch.empty(n, dtype=torch.int32, device="cuda")
    d_n = torch.zeros(1, dtype=torch.int64, device="cuda")
    step = lambda: plan.frontier_device(d_idx.data_ptr(), d_n.data_ptr())  # noqa: E731
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = ctx.lib.pals_ctx_launch_count(ctx.h)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for k in range(args.steps):
        l2_flush()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    launches = ctx.lib.pals_ctx_launch_count(ctx.h) - l0
    t_max = dist.max(float(np.sum([a.elapsed_time(b) for a, b in ev])))
    value = dist.sum(float(n)) * args.steps / (t_max * 1e-3)
    idx = plan.frontier()  # warm-up of the host-output path (its scratch buffer)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        idx = plan.frontier()
    e2e_t = dist.max(time.perf_counter() - t0)
    return {"metric": "frontier points/s (evaluate + build_frontier over a dense grid)",
            "value": value, "unit": "points/s", "ms_per_step": t_max / args.steps,
            "steps": args.steps, "workload": FRONTIER_WORKLOAD, "points_per_gpu": n,
            "frontier_size": int(d_n.item()), "gpu_launches": int(launches),
            "e2e": {"value": dist.sum(float(n)) * args.steps / e2e_t, "unit": "points/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8 + 4 * len(idx),
                    "api": "pals_plan_frontier (C ABI, host index output)"}}


def cpu_frontier(seconds):
    """evaluate + build_frontier through the unmodified reference (sequential by design)."""
    from paper_2605_21427_b200 import workloads
    kind, ref = _reference_backend()
    if kind != "reference":
        return {"value": None, "unit": "points/s", "cores": 0, "kind": "port",
                "sample": "reference build absent"}
    from oracle.oracle import ref_bench_frontier
    c = workloads.cfg3_extended()
    t, _ = ref_bench_frontier(ref, c["profile"], c["gpu"], c["coeffs"], c["points"], 1)
    reps = int(max(1, min(20, seconds / max(t, 1e-3))))
    t, _ = ref_bench_frontier(ref, c["profile"], c["gpu"], c["coeffs"], c["points"], reps)
    n = len(c["points"])
    return {"value": reps * n / t, "unit": "points/s", "cores": 1, "kind": "reference",
            "sample": f"{reps} x the 589,824-point grid through cluster_throughput + "
                      f"efficiency + build_frontier (single-threaded, as evaluate_regime), "
                      f"{t:.1f} s"}


def cpu_allocate(args, seconds):
    """allocate_budget through the unmodified reference, all host threads."""
    from paper_2605_21427_b200 import workloads
    kind, ref = _reference_backend()
    from oracle.oracle import Oracle, oracle_allocate, ref_bench_allocate
    s = workloads.cfg4_setup()
    orc = Oracle()
    tm, pm = [], []
    for p in s["profiles"]:
        pts = workloads.grid_points(s["caps"], s["batches"], [p.deploy_tp], [p.deploy_ep], [1])
        T, P, _ = orc.eval(p, s["gpu"], pts)
        tm.append(float(T.max()))
        pm.append(float((s["coeffs"].alpha * 4 * P + s["coeffs"].beta_watts).max()))
    threads = os.cpu_count() or 1
    if kind == "reference":
        probe = workloads.alloc_problems(2000 * threads, 2605, tm, pm, s["gpu"], s["coeffs"])
        t, _ = ref_bench_allocate(ref, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                  s["batches"], 25.0, 0.02, probe, threads)
        rate = len(probe["budget"]) / t
        n = int(max(2000 * threads, min(args.clusters, rate * seconds)))
        prob = workloads.alloc_problems(n, 2605, tm, pm, s["gpu"], s["coeffs"])
        t, _ = ref_bench_allocate(ref, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                  s["batches"], 25.0, 0.02, prob, threads)
        return {"value": n / t, "unit": "allocations/s", "cores": threads, "kind": "reference",
                "sample": f"{n} clusters of the same workload through the unmodified "
                          f"allocate_budget (analytic scorer, steps rebuilt per call as the "
                          f"reference does), {threads} threads, {t:.1f} s"}
    prob = workloads.alloc_problems(2000, 2605, tm, pm, s["gpu"], s["coeffs"])
    t0 = time.perf_counter()
    oracle_allocate(orc, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], 25.0,
                    0.02, prob)
    t = time.perf_counter() - t0
    return {"value": 2000 / t, "unit": "allocations/s", "cores": 1, "kind": "port",
            "sample": "2000 clusters, C restatement, 1 thread"}


# ---------------------------------------------------------- CPU reference --
def _reference_backend():
    """The reference build (oracle/_ref) when present, else the C restatement."""
    from oracle.oracle import Oracle, Reference
    if Reference.available():
        return "reference", Reference()
    return "port", Oracle()


def issue_roofline(kernel, units_per_s, unit, clk, note):
    """A latency / issue-bound kernel against instruction issue (one warp instruction per SMSP
    per cycle): warp instructions per unit from the committed ncu capture of this build at the
    bench size (smsp__inst_executed over the capture's units) x the live unit rate, over the
    issue peak at the sampled SM clock. Also reports ncu's issue-active share."""
    inst = ncu_metric(kernel, "warp_inst")
    units = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "capture_sizes.json")) as f:
            units = json.load(f)[kernel]["units"]
    except Exception:
        pass
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak = 148 * 4 * mhz * 1e6
    if not inst or not units:
        return {"bound": "issue", "kernel": kernel, "achieved": None, "peak": peak / 1e9,
                "unit": "G warp-instructions/s", "frac": None, "traffic": ncu_traffic(kernel),
                "note": "no committed ncu capture for this build"}
    per = inst / units
    ach = per * units_per_s
    return {"bound": "issue", "kernel": kernel, "achieved": ach / 1e9, "peak": peak / 1e9,
            "unit": "G warp-instructions/s", "frac": ach / peak, "traffic": ncu_traffic(kernel),
            "warp_instructions_per_" + unit.rstrip("s"): per,
            "issue_active_pct_ncu": ncu_metric(kernel, "issue_active_pct"),
            "peak_source": f"1 warp instruction / SMSP / cycle x 4 x 148 SMs at {mhz:.0f} MHz "
                           "(sampled); instructions per unit from profiles/ncu_summary.json",
            "algorithmic": note}


def decide_leg(args, dist, plan, d_q, nq, h_qn, stream, l2_flush, ref_pairs_per_s, n_cfg):
    """Time to decide the same queries with the prefix-min path (PALS_DECIDE_PREFIX, same
    decisions as the pair scan): device step time and end to end through pals_select with
    pinned host buffers; queries/s beside the reference's queries/s (its config evals/s over
    the grid size)."""
    import torch
    from paper_2605_21427_b200.abi import ptr
    d_i = torch.empty(nq, dtype=torch.int32, device="cuda")
    d_r = torch.empty(nq, dtype=torch.uint8, device="cuda")
    h_i = torch.empty(nq, dtype=torch.int32, pin_memory=True).numpy()
    h_r = torch.empty(nq, dtype=torch.uint8, pin_memory=True).numpy()
    plan.time_scan(False)
    plan.set_decide("prefix")
    lib = plan.ctx.lib
    try:
        run = lambda: plan.run(d_q.data_ptr(), nq, d_i.data_ptr(), d_r.data_ptr())  # noqa
        for _ in range(max(1, args.warmup)):
            run()
        torch.cuda.synchronize()
        ms = []
        for _ in range(args.steps):
            l2_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = dist.max(float(np.mean(ms)))

        def e2e():
            rc = lib.pals_select(plan.h, ptr(h_qn), nq, ptr(h_i), ptr(h_r))
            assert rc == 0, lib.pals_last_error()

        e2e()
        em = []
        for _ in range(args.steps):
            l2_flush()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e()
            e1.record(stream)
            e1.synchronize()
            em.append(e0.elapsed_time(e1))
        te = dist.max(float(np.mean(em)))
    finally:
        plan.set_decide("scan")
    total_q = dist.sum(float(nq))
    out = {"api": "PALS_DECIDE_PREFIX: prefix-min tables instead of the pair scan, the same "
                  "decisions (tests/test_gpu_select.py)",
           "ms_per_step": t, "queries_per_s": total_q / (t * 1e-3),
           "e2e": {"queries_per_s": total_q / (te * 1e-3), "ms_per_step": te,
                   "h2d_bytes_per_step": nq * 48, "d2h_bytes_per_step": nq * 5}}
    if ref_pairs_per_s:
        ref_qps = ref_pairs_per_s / n_cfg
        out["reference_queries_per_s"] = ref_qps
        out["e2e_speedup_vs_reference"] = out["e2e"]["queries_per_s"] / ref_qps
    return out


def scan_mix():
    """ALU-pipe warp instructions per (config, query) pair per thread of the pair-scan loops,
    from the committed SASS analysis (scripts/sass_mix.py) of the build being measured."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "k_scan_mix.json")) as f:
            m = json.load(f)["alu_warp_inst_per_pair_lane"]
        return float(m["A/C"]), float(m["B"]), "profiles/r02/k_scan_mix.json"
    except Exception:
        return 1.5, 3.5, "built-in (LOP3 + 1/2 VIMNMX3 per A/C pair; 2 LOP3 + VIADDMNMX + 1/2 VIMNMX3 per B pair)"


def scan_roofline(counts, n_cfg, scan_ms, clk):
    """k_scan against the ALU pipe, the resource its instruction mix binds: ALU lane
    operations issued per second (from the SASS mix x the pairs actually scanned) over the
    ALU pipe's peak (16 lanes per SMSP, 4 SMSPs x 148 SMs at the SM clock sampled during
    the run)."""
    a_c, b, src = scan_mix()
    pairs_ac = float(counts[0] + counts[2]) * n_cfg
    pairs_b = float(counts[1]) * n_cfg
    alu_ops = a_c * pairs_ac + b * pairs_b  # lane operations on the ALU pipe
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak = 148 * 4 * 16 * mhz * 1e6
    achieved = alu_ops / (scan_ms * 1e-3)
    return {"bound": "alu", "kernel": "k_scan", "achieved": achieved / 1e12, "peak": peak / 1e12,
            "unit": "Tops/s (ALU-pipe lane ops)", "frac": achieved / peak,
            "traffic": ncu_traffic("k_scan"),
            "pairs_per_s": (pairs_ac + pairs_b) / (scan_ms * 1e-3),
            "algorithmic": "per scanned (config, query) pair: one feasibility compare and one "
                           "argmin update (two per side for QoS+budget queries), executed as "
                           f"{a_c} ALU-pipe instructions per pair (classes A/C) and {b} (class B) "
                           "plus one FMA-pipe IMAD.IADD per side",
            "peak_source": f"B200 ALU pipe 16 lanes/SMSP x 4 x 148 SMs at {mhz:.0f} MHz "
                           f"(sampled); instruction mix from {src}",
            "ncu_alu_pipe_pct_of_active": ncu_metric("k_scan", "alu_pipe_pct")}


def select_config_dict(args, world, n_cfg=65_536):
    """The headline workload's config, identical in both arms (the driver compares them)."""
    return {"workload": SELECT_WORKLOAD, "queries_per_gpu": args.queries, "configs": n_cfg,
            "global_batch": args.queries * world, "parallelism": f"shard{world}",
            "l2": "flushed between GPU steps (256 MiB device write)"}


def parity_of(got, want, against="oracle/_ref (the unmodified reference headers)"):
    """{checked, mismatches, against}: element-wise (per record, all bytes) comparison."""
    got = np.ascontiguousarray(got)
    want = np.ascontiguousarray(want)
    n = min(len(got), len(want))
    g = got[:n].view(np.uint8).reshape(n, -1)
    w = want[:n].view(np.uint8).reshape(n, -1)
    return {"checked": int(n), "mismatches": int((g != w).any(1).sum()), "against": against}


def cpu_select(args, cfg, tref, seconds, results=None):
    """select_config + analytic_scorer over cfg2 queries on all host threads. `results`
    (a dict) receives the reference's decisions for the timed sample."""
    from paper_2605_21427_b200 import workloads
    kind, ref = _reference_backend()
    threads = os.cpu_count() or 1
    n = len(cfg["points"])
    if kind == "reference":
        q = workloads.gen_queries(max(threads, 4 * threads), cfg["seed"], tref, "qos")
        t, _, _ = ref.bench_select(cfg["profile"], cfg["gpu"], cfg["points"], cfg["coeffs"], q,
                                   threads, want_results=False)
        rate = len(q) * n / t
        nq = int(min(args.queries, max(threads, rate * seconds / n)))
        q = workloads.gen_queries(nq, cfg["seed"], tref, "qos")
        t, ri, rr = ref.bench_select(cfg["profile"], cfg["gpu"], cfg["points"], cfg["coeffs"], q,
                                     threads, want_results=results is not None)
        if results is not None:
            results.update(index=ri, reason=rr)
        return {"value": nq * n / t, "unit": "config evals/s", "cores": threads,
                "kind": "reference",
                "sample": f"{nq} cfg2 queries x {n} configs through the unmodified "
                          f"select_config+analytic_scorer, {threads} threads, {t:.1f} s"}
    # the C port is single threaded
    T, P, _ = ref.eval(cfg["profile"], cfg["gpu"], cfg["points"])
    q = workloads.gen_queries(50, cfg["seed"], tref, "qos")
    t0 = time.perf_counter()
    ref.select(cfg["points"], T, P, cfg["coeffs"], q)
    t = time.perf_counter() - t0
    return {"value": len(q) * n / t, "unit": "config evals/s", "cores": 1, "kind": "port",
            "sample": f"{len(q)} cfg2 queries, C restatement, 1 thread"}


def cpu_replay(args, seconds, results=None):
    from paper_2605_21427_b200 import workloads
    kind, ref = _reference_backend()
    s = workloads.cfg4_setup()
    threads = os.cpu_count() or 1
    if kind == "reference":
        probe = workloads.replay_spec(threads * 4, n_steps=args.trace_steps, seed=2605)
        t, _ = ref.bench_replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                                s["cfg"], probe, threads)
        rate = probe.n_traces * args.trace_steps / t
        ntr = int(max(threads, min(args.traces, rate * seconds / args.trace_steps)))
        spec = workloads.replay_spec(ntr, n_steps=args.trace_steps, seed=2605)
        t, summ = ref.bench_replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                                   s["cfg"], spec, threads)
        if results is not None:
            results["summaries"] = summ
        return {"value": ntr * args.trace_steps / t, "unit": "decisions/s", "cores": threads,
                "kind": "reference",
                "sample": f"{ntr} cfg4 traces x {args.trace_steps} steps through the unmodified "
                          f"control_step (detail::cached analytic scorer), {threads} threads, "
                          f"{t:.1f} s"}
    spec = workloads.replay_spec(8, n_steps=args.trace_steps, seed=2605)
    t0 = time.perf_counter()
    ref.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], s["cfg"], spec)
    t = time.perf_counter() - t0
    return {"value": 8 * args.trace_steps / t, "unit": "decisions/s", "cores": 1, "kind": "port",
            "sample": f"8 cfg4 traces, C restatement, 1 thread"}


def cpu_predict(args, bundle, seconds):
    """PredictorBundle::predict on all host threads (the reference build)."""
    from paper_2605_21427_b200 import workloads
    kind, ref = _reference_backend()
    if kind != "reference":
        return {"value": None, "unit": "predictions/s", "cores": 0, "kind": "port",
                "sample": "reference build absent"}
    from oracle.oracle import ref_bench_predict
    threads = os.cpu_count() or 1
    path = os.path.join(tempfile.gettempdir(), "pals_bench_bundle.json")
    bundle.to_json(path)
    pts = workloads.predict_points(20_000 * threads, seed=2605)
    t = ref_bench_predict(ref, path, "mixtral-8x7b-like", pts, threads)
    rate = len(pts) / t
    n = int(min(2_000_000 * threads, max(len(pts), rate * seconds)))
    pts = workloads.predict_points(n, seed=2605)
    t = ref_bench_predict(ref, path, "mixtral-8x7b-like", pts, threads)
    return {"value": n / t, "unit": "predictions/s", "cores": threads, "kind": "reference",
            "sample": f"{n} random points through the unmodified PredictorBundle::predict "
                      f"(same bundle), {threads} threads, {t:.1f} s"}


def cpu_latency(c1, tmax):
    """One select_config call on the cfg1 grid through the unmodified reference (1 thread)."""
    kind, ref = _reference_backend()
    if kind != "reference":
        return None
    from paper_2605_21427_b200.wattserve import make_queries
    q = make_queries(np.full(20_000, 0.6 * tmax), 1600.0, 1.0, 0.05, 0.02)
    t, _, _ = ref.bench_select(c1["profile"], c1["gpu"], c1["points"], c1["coeffs"], q, 1,
                               want_results=False)
    return t / len(q) * 1e6


def run_reference(args, dist: Dist):
    """The reference's own CPU implementation of the path, all host threads, rank 0."""
    if dist.rank != 0:
        return
    from paper_2605_21427_b200 import workloads
    from oracle.oracle import Reference
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libwsref.so not built (needs /root/reference at build)"}))
        return
    cfg = workloads.cfg2(args.queries)
    ref = Reference()
    T, P, _ = ref.eval(cfg["profile"], cfg["gpu"], cfg["points"])
    tref = float(np.max(T * cfg["points"]["dp"]))
    per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    vals = []
    for k in range(args.warmup + args.steps):
        b = cpu_select(args, cfg, tref, per_step)
        if k >= args.warmup:
            vals.append(b)
    v = float(np.mean([b["value"] for b in vals]))
    dec = cpu_replay(args, per_step)
    alc = cpu_allocate(args, per_step)
    fro = cpu_frontier(per_step)
    c3 = workloads.cfg3(args.cfg3_queries)
    T3, _, _ = ref.eval(c3["profile"], c3["gpu"], c3["points"])
    s3 = cpu_cfg3(args, c3, float(np.max(T3 * c3["points"]["dp"])), per_step)
    sm = cpu_sim(args, per_step) if args.sim_seeds > 0 else None
    from paper_2605_21427_b200.forest import Bundle
    pr = cpu_predict(args, Bundle.load_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data",
                                                        "predictor_default.npz")), per_step)
    zero = {"h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "config evals/s",
           "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": select_config_dict(args, dist.world, len(cfg["points"])),
           "cpu_baseline": vals[-1],
           "e2e": {"value": v, "unit": "config evals/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "decisions": {"metric": "controller decisions/s", "value": dec["value"],
                         "unit": "decisions/s", "workload": REPLAY_WORKLOAD,
                         "cpu_baseline": dec,
                         "e2e": {"value": dec["value"], "unit": "decisions/s",
                                 "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}},
           "predictions": {"metric": "predictor predictions/s (PredictorBundle::predict, T "
                                     "and P)", "value": pr["value"], "unit": "predictions/s",
                           "cpu_baseline": pr,
                           "e2e": {"value": pr["value"], "unit": "predictions/s", **zero}},
           "frontiers": {"metric": "frontier points/s", "value": fro["value"],
                         "unit": "points/s", "workload": FRONTIER_WORKLOAD,
                         "cpu_baseline": fro,
                         "e2e": {"value": fro["value"], "unit": "points/s",
                                 "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}},
           "allocations": {"metric": "cluster budget allocations/s", "value": alc["value"],
                           "unit": "allocations/s", "workload": ALLOC_WORKLOAD,
                           "cpu_baseline": alc,
                           "e2e": {"value": alc["value"], "unit": "allocations/s",
                                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}},
           "cfg3": {"metric": "config evals/s (cfg3 select_config, MoE grid, mixed QoS/budget "
                              "queries)", "value": s3["value"], "unit": "config evals/s",
                    "workload": CFG3_WORKLOAD, "cpu_baseline": s3,
                    "e2e": {"value": s3["value"], "unit": "config evals/s", **zero}},
           "cfg5": {"metric": "controller decisions/s (cfg5, strong scaling over the GPUs)",
                    "value": dec["value"], "unit": "decisions/s", "workload": CFG5_WORKLOAD,
                    "cpu_baseline": dec,
                    "e2e": {"value": dec["value"], "unit": "decisions/s", **zero}},
           "scenarios": None if sm is None else {
               "metric": "scenario node-intervals/s (run_scenario queue plant, 5-policy suites)",
               "value": sm["value"], "unit": "node-intervals/s", "workload": SIM_WORKLOAD,
               "cpu_baseline": sm, "e2e": {"value": sm["value"], "unit": "node-intervals/s",
                                           **zero}}}
    print(json.dumps(out), flush=True)


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: launch the N ranks here (one process
    per GPU, torchrun rendezvous on 127.0.0.1) instead of silently measuring one GPU."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        spawn_ranks(args)  # does not return
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
    else:
        run_ours(args, dist)


if __name__ == "__main__":
    main()
