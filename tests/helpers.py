"""Shared drivers so the oracle and the GPU path are checked by the same code."""
from __future__ import annotations

import numpy as np

from paper_2605_21427_b200 import abi
from paper_2605_21427_b200.abi import CtrlState, Telemetry, default_ctrl_cfg
from paper_2605_21427_b200.wattserve import make_targets


def ladder(n, t_lo, t_hi):
    """TableScorer ladder of tests/test_controller.cpp:31-43."""
    pts = np.zeros(n, abi.POINT_DT)
    T = np.zeros(n)
    P = np.zeros(n)
    for i in range(n):
        frac = 0.0 if n == 1 else i / (n - 1)
        thr = t_lo + (t_hi - t_lo) * frac
        pts[i] = (150.0 + i, 1 + i, 2, 1, 1)
        T[i] = thr
        P[i] = 40.0 + thr * thr / 800.0
    return pts, T, P


def first_match(pts):
    """canon[i] = first index whose point equals pts[i] (OperatingPoint::operator==)."""
    canon = np.arange(len(pts))
    seen = {}
    for i, p in enumerate(pts.tolist()):
        canon[i] = seen.setdefault(tuple(p), i)
    return canon


def table_view(pts, T, P):
    """What TableScorer returns per candidate (first match by value) and the canon map."""
    c = first_match(pts)
    return T[c], P[c], c


def table_cases(gold):
    t = gold("tables")
    off, qoff = t["off"], t["qoff"]
    for c in range(len(off) - 1):
        yield (t["points"][off[c]:off[c + 1]], t["T"][off[c]:off[c + 1]],
               t["P"][off[c]:off[c + 1]], t["queries"][qoff[c]:qoff[c + 1]],
               t["idx"][qoff[c]:qoff[c + 1]], t["reason"][qoff[c]:qoff[c + 1]])


def run_control_sequences(gold, step_fn, max_seqs=None):
    """Re-drive the recorded control_step sequences (tests/golden/control.npz) through
    step_fn(pts, T, P, tel, now, targets, state, cfg) -> (decision, state); returns the
    list of mismatching (seq, k, field) tuples."""
    g = gold("control")
    steps, seqs = g["steps"], g["seqs"]
    bad = []
    for sq in seqs[:max_seqs]:
        pts, T, P = ladder(int(sq["n"]), 300.0, 2400.0)
        cfg = default_ctrl_cfg(target_headroom=float(sq["headroom"]),
                               budget_margin=float(sq["margin"]))
        st = CtrlState()
        st.bias = 1.0
        st.current = abi.Point(*pts[-1].tolist())
        for r in steps[steps["seq"] == sq["seq"]]:
            b = None if np.isnan(r["budget"]) else float(r["budget"])
            tg = make_targets(float(r["tps"]), b, 0.05, int(r["objective"]))
            # the recorded measurement that the reference saw at this step
            k = int(r["k"])
            prev = steps[(steps["seq"] == sq["seq"]) & (steps["k"] == k - 1)]
            measured = (float(prev["measured"][0]) if k > 0
                        else float(sq["lam"]) * float(T[-1]))
            tel = Telemetry(float(r["t_s"]), measured)
            d, st = step_fn(pts, T, P, tel, float(r["now"]), tg, st, cfg)
            got = (d.point.cap_watts, d.point.batch, d.applied, d.reason, st.bias, st.integral,
                   st.prev_error, st.has_prev_error, st.sustain_count, st.current.cap_watts,
                   st.current.batch)
            want = (r["d_cap"], r["d_batch"], r["applied"], r["reason"], r["bias"],
                    r["integral"], r["prev_error"], r["has_prev"], r["sustain"], r["cur_cap"],
                    r["cur_batch"])
            for name, a, w in zip(("cap", "batch", "applied", "reason", "bias", "integral",
                                   "prev_error", "has_prev", "sustain", "cur_cap", "cur_batch"),
                                  got, want):
                if not (a == w or (isinstance(a, float) and np.isnan(a) and np.isnan(w))):
                    bad.append((int(sq["seq"]), k, name, a, w))
    return bad


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


# ---- allocate_budget (allocator.hpp) restated in Python for small cases --------------
def py_steps(T, P, cdp, alpha, beta, margin=0.0):
    """detail::throughput_steps (allocator.hpp:34-56) + the margin scaling (:106)."""
    pts = [(float(d) * (alpha * 4 * float(p) + beta), float(d) * float(t))
           for t, p, d in zip(T, P, cdp)]
    pts.sort(key=lambda s: (s[0], -s[1]))
    steps, best = [], 0.0
    for pw, th in pts:
        if th > best + 1e-12:
            steps.append([pw, th])
            best = th
    for s in steps:
        s[0] /= 1.0 - margin
    return steps


def py_allocate(steps, dps, targets, budget, floor_unit, quantum=25.0):
    """allocate_budget (allocator.hpp:76-186) over precomputed steps; None = config_error."""
    import math
    n = len(steps)
    if n == 0:
        return None
    floors = [float(d) * floor_unit for d in dps]
    ft = 0.0
    for f in floors:
        ft += f
    if ft > budget:
        return None
    bud = list(floors)
    rem = budget - ft

    def under(st, b):
        best = 0.0
        for pw, th in st:
            if pw > b:
                break
            best = th
        return best

    cur = [under(steps[i], bud[i]) for i in range(n)]
    while rem >= quantum:
        unmet = any(not (cur[i] >= targets[i]) for i in range(n))
        br, bc, bi = 0.0, 0.0, n
        for i in range(n):
            if unmet and cur[i] >= targets[i]:
                continue
            for pw, th in steps[i]:
                if pw <= bud[i] or th <= cur[i]:
                    continue
                cost = math.ceil((pw - bud[i]) / quantum) * quantum
                if cost > rem:
                    break
                gain = (min(th, targets[i]) - min(cur[i], targets[i])) if unmet else th - cur[i]
                if gain <= 1e-12:
                    continue
                rate = gain / cost
                if bi == n or rate > br + 1e-12 or (rate > br - 1e-12 and bud[i] < bud[bi] - 1e-12):
                    br, bc, bi = rate, cost, i
        if bi == n:
            break
        bud[bi] += bc
        cur[bi] = under(steps[bi], bud[bi])
        rem -= bc
    ceil_ = [bud[i] if not steps[i] else steps[i][-1][0] + 2.0 * quantum for i in range(n)]
    while rem >= quantum:
        lo = n
        for i in range(n):
            if bud[i] + quantum > ceil_[i]:
                continue
            if lo == n or bud[i] < bud[lo]:
                lo = i
        if lo == n:
            break
        bud[lo] += quantum
        rem -= quantum
    tot = 0.0
    for b in bud:
        tot += b
    return bud, tot, all(cur[i] >= targets[i] for i in range(n))


def alloc_setup(oracle):
    """cfg4's 8 profiles at their deployments with dp = 1: unconstrained throughput and
    peak node power per model (scales for workloads.alloc_problems)."""
    from paper_2605_21427_b200 import workloads
    s = workloads.cfg4_setup()
    tm, pm = [], []
    for p in s["profiles"]:
        pts = workloads.grid_points(s["caps"], s["batches"], [p.deploy_tp], [p.deploy_ep], [1])
        T, P, _ = oracle.eval(p, s["gpu"], pts)
        tm.append(float(T.max()))
        pm.append(float((s["coeffs"].alpha * 4 * P + s["coeffs"].beta_watts).max()))
    s["t_max"], s["p_max"] = tm, pm
    return s
