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
