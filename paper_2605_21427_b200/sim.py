"""Batched queue-plant scenario simulation (K6): the reference's run_scenario /
run_baseline_suite (sim.hpp:482-500) on the GPU through pals_run_scenarios.

Scenario files use the reference's schema (scenario_io.hpp:35-93); the bundled
scenarios ship as data/scenarios.json (re-emitted from the reference's
proj/data/scenarios + traces by oracle/gen_golden.py). Results mirror the
reference's SimResult logs and RunSummary (metrics.hpp:24-102); telemetry_csv /
decisions_csv format them byte-for-byte like metrics.hpp:130-157.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from .abi import (OBJ_BUDGET, OBJ_QOS, POLICIES, REASON_NAMES, SIM_DEC_DT, SIM_NODE_RESULT_DT,
                  SIM_REQ_DT, SIM_RESULT_DT, SIM_TEL_DT, CtrlCfg, Profile, Scenario, SimNode,
                  default_ctrl_cfg, ptr)
from ._lib import check

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "scenarios.json")
POLICY_NAMES = {v: k for k, v in POLICIES.items()}


def scenario_from_dict(j: dict, trace=None) -> dict:
    """scenario_from_json (scenario_io.hpp:35-93): defaults as the reference applies them.
    `trace` = [(t_s, watts), ...] (the loaded budget_trace_csv), or None."""
    sc = {"name": j["name"], "duration_s": float(j["duration_s"]),
          "interval_s": float(j.get("interval_s", 0.5)), "seed": int(j["seed"]),
          "mean_tokens": 200.0, "log_sigma": 0.4, "cluster_budget_w": None, "trace": trace or [],
          "policy": j.get("policy", "joint"), "objective": j.get("objective", "qos")}
    if "output_tokens" in j:
        sc["mean_tokens"] = float(j["output_tokens"]["mean"])
        sc["log_sigma"] = float(j["output_tokens"]["log_sigma"])
    if j.get("cluster_budget_w") is not None:
        sc["cluster_budget_w"] = float(j["cluster_budget_w"])
    if sc["policy"] not in POLICIES:
        raise ValueError("unknown policy: " + sc["policy"])
    if sc["objective"] not in ("qos", "budget-throughput"):
        raise ValueError("unknown objective: " + sc["objective"])
    c = j.get("controller")
    if c is not None:
        sc["epsilon"] = float(c.get("epsilon", 0.05))
        sc["controller"] = dict(kp=float(c.get("kp", 0.5)), ki=float(c.get("ki", 0.1)),
                                kd=float(c.get("kd", 0.05)),
                                sustain_intervals=int(c.get("sustain_intervals", 3)),
                                integral_clamp=float(c.get("integral_clamp", 0.5)),
                                target_headroom=float(c.get("headroom", sc["epsilon"])),
                                budget_margin=float(c.get("budget_margin", 0.02)))
    else:
        sc["epsilon"] = 0.05
        sc["controller"] = dict(target_headroom=0.05, budget_margin=0.02)
    cand = j.get("candidates", {"caps_w": [150, 200, 250, 300, 350, 400],
                                "batches": [1, 4, 8, 16, 32, 64]})
    sc["caps"] = [float(x) for x in cand["caps_w"]]
    sc["batches"] = [int(x) for x in cand["batches"]]
    if "initial" in j:
        sc["initial_cap_w"] = float(j["initial"]["cap_w"])
        sc["initial_batch"] = int(j["initial"]["batch"])
    else:
        sc["initial_cap_w"] = max(sc["caps"])
        sc["initial_batch"] = max(sc["batches"])
    sc["nodes"] = [dict(model=n["model"], qos_fraction=float(n.get("qos_fraction", 1.0)),
                        tp=int(n.get("tp", 1)), ep=int(n.get("ep", 1)), dp=int(n.get("dp", 1)),
                        arrival_rate_per_s=float(n["arrival_rate_per_s"]),
                        initial_backlog=int(n.get("initial_backlog", 0)))
                   for n in j["nodes"]]
    return sc


def bundled_scenarios(path: str = DATA) -> dict:
    """The reference's three bundled scenarios: single_node, multinode_qos,
    demand_response (proj/data/scenarios/*.json, traces resolved)."""
    with open(path) as f:
        j = json.load(f)
    return {k: scenario_from_dict(v["scenario"], [tuple(x) for x in v["trace"]] or None)
            for k, v in j.items()}


class _CScenario:
    """A pals_scenario plus the arrays it points to (kept alive together)."""

    def __init__(self, sc: dict, model_index: dict, memo: dict | None = None):
        # memo: arrays and controller configs shared by the scenarios of one call (a seed
        # sweep repeats the same candidate axes, traces and controller for every seed)
        memo = {} if memo is None else memo

        def shared(key, make):
            v = memo.get(key)
            if v is None:
                v = memo[key] = make()
            return v

        self.caps = shared(("caps", id(sc["caps"])),
                           lambda: np.ascontiguousarray(sc["caps"], np.float64))
        self.batches = shared(("batches", id(sc["batches"])),
                              lambda: np.ascontiguousarray(sc["batches"], np.int32))

        def split_trace():
            tr = np.asarray(sc["trace"], np.float64).reshape(-1, 2)
            return np.ascontiguousarray(tr[:, 0]), np.ascontiguousarray(tr[:, 1])

        self.tt, self.tw = shared(("trace", id(sc["trace"])), split_trace)
        def make_nodes():
            nodes = (SimNode * len(sc["nodes"]))()
            for i, n in enumerate(sc["nodes"]):
                nodes[i] = SimNode(model_index[n["model"]], n["tp"], n["ep"], n["dp"],
                                   n["qos_fraction"], n["arrival_rate_per_s"],
                                   n["initial_backlog"], 0)
            return nodes

        self.nodes = shared(("nodes", id(sc["nodes"])), make_nodes)
        s = Scenario()
        s.duration_s, s.interval_s, s.seed = sc["duration_s"], sc["interval_s"], sc["seed"]
        s.mean_tokens, s.log_sigma = sc["mean_tokens"], sc["log_sigma"]
        s.has_cluster_budget = 1 if sc["cluster_budget_w"] is not None else 0
        s.cluster_budget_w = sc["cluster_budget_w"] or 0.0
        s.n_trace = len(self.tt)
        s.trace_t = self.tt.ctypes.data if len(self.tt) else None
        s.trace_w = self.tw.ctypes.data if len(self.tw) else None
        s.policy = POLICIES[sc["policy"]]
        s.objective = OBJ_QOS if sc["objective"] == "qos" else OBJ_BUDGET
        ck = ("ctrl",) + tuple(sorted(sc["controller"].items()))
        s.controller = shared(ck, lambda: default_ctrl_cfg(**sc["controller"]))
        s.epsilon = sc["epsilon"]
        s.cand_caps = self.caps.ctypes.data
        s.cand_batches = self.batches.ctypes.data
        s.n_caps, s.n_batches = len(self.caps), len(self.batches)
        s.initial_cap_w, s.initial_batch = sc["initial_cap_w"], sc["initial_batch"]
        s.n_nodes = len(sc["nodes"])
        s.nodes = C.addressof(self.nodes)
        self.c = s


def _model_index(profiles):
    return {p.name.decode(): i for i, p in enumerate(profiles)}


def n_intervals(sc: dict) -> int:
    """sim.hpp:224: llround(duration / interval)."""
    x = sc["duration_s"] / sc["interval_s"]
    return int(np.floor(x + 0.5)) if x >= 0 else -int(np.floor(-x + 0.5))


def run_scenarios(ctx, scenarios, profiles, gpu, coeffs, predictors=None, logs: bool = False,
                  requests: bool = False):
    """run_scenario for every scenario dict (policy etc. inside each) on the GPU.
    predictors: {model_name: forest model handle} (predictor_scorer) or None.
    Returns (node_results, results, telemetry, decisions): node_results is
    SIM_NODE_RESULT_DT in scenario/node order; with logs, telemetry / decisions are
    [total_nodes, max_intervals] arrays of SIM_TEL_DT / SIM_DEC_DT."""
    idx = _model_index(profiles)
    memo: dict = {}
    cs = [_CScenario(s, idx, memo) for s in scenarios]
    arr = (Scenario * len(cs))(*[c.c for c in cs])
    profs = (Profile * len(profiles))(*profiles)
    preds = (C.c_void_p * len(profiles))()
    for name, m in (predictors or {}).items():
        preds[idx[name]] = m.h
    n_nodes = sum(len(s["nodes"]) for s in scenarios)
    stride = max(n_intervals(s) for s in scenarios) if logs else 0
    nres = np.zeros(n_nodes, SIM_NODE_RESULT_DT)
    res = np.zeros(len(cs), SIM_RESULT_DT)
    tel = np.zeros((n_nodes, max(stride, 1)), SIM_TEL_DT) if logs else None
    dec = np.zeros((n_nodes, max(stride, 1)), SIM_DEC_DT) if logs else None
    check(ctx.lib.pals_sim_keep_requests(ctx.h, 1 if requests else 0))
    check(ctx.lib.pals_run_scenarios(ctx.h, len(cs), arr, len(profiles), profs, preds,
                                     C.byref(gpu), C.byref(coeffs), ptr(nres), ptr(res), stride,
                                     ptr(tel), ptr(dec)))
    if not requests:
        return nres, res, tel, dec
    reqs = []
    for i in range(n_nodes):
        n = C.c_int64(0)
        check(ctx.lib.pals_sim_requests(ctx.h, i, None, 0, C.byref(n)))
        r = np.zeros(n.value, SIM_REQ_DT)
        check(ctx.lib.pals_sim_requests(ctx.h, i, ptr(r), n.value, C.byref(n)))
        reqs.append(r)
    check(ctx.lib.pals_sim_keep_requests(ctx.h, 0))
    return nres, res, tel, dec, reqs


def last_timing(ctx):
    """(host setup seconds, simulation kernel ms) of the last run_scenarios on ctx."""
    a, b = C.c_double(), C.c_double()
    check(ctx.lib.pals_sim_last_timing(ctx.h, C.byref(a), C.byref(b)))
    return a.value, b.value


def run_baseline_suite(ctx, scenario, profiles, gpu, coeffs, predictors=None, logs=False):
    """All five policies on identical arrival streams (sim.hpp:488-500)."""
    scs = [dict(scenario, policy=p) for p in POLICIES]
    return dict(zip(POLICIES, _split(run_scenarios(ctx, scs, profiles, gpu, coeffs, predictors,
                                                   logs), scs)))


def _split(out, scs):
    nres, res, tel, dec = out
    parts, o = [], 0
    for i, s in enumerate(scs):
        k = len(s["nodes"])
        parts.append((nres[o:o + k], res[i], None if tel is None else tel[o:o + k],
                      None if dec is None else dec[o:o + k]))
        o += k
    return parts


def _g(v: float) -> str:
    return "%.10g" % v  # fmt_num (csvio.hpp:17-21)


def telemetry_csv(scenario: dict, tel: np.ndarray) -> bytes:
    """telemetry_csv (metrics.hpp:130-143) of one scenario's [nodes, intervals] log."""
    n = n_intervals(scenario)
    out = ["node,model,t_s,gpu_power_w,sys_power_w,throughput_tps,utilization,queue_depth,"
           "active_batch,node_budget_w,applied_cap_w,applied_batch_cap\n"]
    for i, nd in enumerate(scenario["nodes"]):
        for t in tel[i, :n]:
            out.append(f"{i},{nd['model']},{_g(t['t_s'])},{_g(t['gpu_power_w'])},"
                       f"{_g(t['sys_power_w'])},{_g(t['throughput_tps'])},{_g(t['utilization'])},"
                       f"{int(t['queue_depth'])},{int(t['active_batch'])},"
                       f"{_g(t['node_budget_w'])},{_g(t['applied_cap_w'])},"
                       f"{int(t['applied_batch_cap'])}\n")
    return "".join(out).encode()


def decisions_csv(scenario: dict, tel: np.ndarray, dec: np.ndarray) -> bytes:
    """decisions_csv (metrics.hpp:145-157) of one scenario's [nodes, intervals] log."""
    n = n_intervals(scenario)
    out = ["node,model,t_s,cap_w,batch,tp,ep,dp,applied,reason,err_norm,bias\n"]
    for i, nd in enumerate(scenario["nodes"]):
        for t, d in zip(tel[i, :n], dec[i, :n]):
            out.append(f"{i},{nd['model']},{_g(t['t_s'])},{_g(d['cap_w'])},{int(d['batch'])},"
                       f"{nd['tp']},{nd['ep']},{nd['dp']},{int(d['applied'])},"
                       f"{REASON_NAMES[int(d['reason'])]},{_g(d['err_norm'])},{_g(d['bias'])}\n")
    return "".join(out).encode()


def requests_csv(scenario: dict, reqs) -> bytes:
    """requests_csv (metrics.hpp:159-166) from the per-node request records."""
    out = ["node,model,id,arrival_s,output_tokens,generated,completed_s\n"]
    for i, nd in enumerate(scenario["nodes"]):
        m = nd["model"]
        out.extend(f"{i},{m},{int(q['id'])},{_g(q['arrival_s'])},{int(q['output_tokens'])},"
                   f"{_g(q['generated'])},{_g(q['completed_s'])}\n" for q in reqs[i])
    return "".join(out).encode()


__all__ = ["scenario_from_dict", "bundled_scenarios", "run_scenarios", "run_baseline_suite",
           "telemetry_csv", "decisions_csv", "requests_csv", "n_intervals", "CtrlCfg"]
