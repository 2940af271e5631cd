"""TEST INFRASTRUCTURE — regenerate the committed fixtures from the reference.

Runs only in the build container (needs /root/reference and oracle/_ref):
  python oracle/gen_golden.py

Writes
  paper_2605_21427_b200/data/profiles.json  the reference's calibrated model-fit
      inputs (proj/data/profiles/*.json + platform.json), loaded through the
      reference's own nlohmann loader (json_io.hpp:70-105) and re-emitted with
      repr()-exact doubles;
  tests/golden/*.npz  outputs of the UNMODIFIED reference (oracle/_ref/libwsref.so)
      on seeded inputs: model evaluations, select_config decisions over the
      configs and adversarial near-tie tables, control_step sequences, and
      fluid-plant replays.
"""
from __future__ import annotations

import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2605_21427_b200 import abi, workloads  # noqa: E402
from paper_2605_21427_b200.abi import (POINT_DT, QUERY_DT, STEPLOG_DT, CtrlState,  # noqa: E402
                                       Telemetry)
from paper_2605_21427_b200.profiles import load_bundle  # noqa: E402

REF_DATA = "/root/reference/proj/data"
GOLD = os.path.join(ROOT, "tests", "golden")


def profile_to_dict(p) -> dict:
    d = {k: getattr(p, k) for k in (
        "compute_fixed", "compute_per_seq", "comm_per_seq", "internode_factor", "knee_watts",
        "compute_power_base", "compute_power_per_seq", "comm_power", "overlap",
        "total_params_b", "active_params_b")}
    d["name"] = p.name.decode()
    d["comm_fixed_by_tp"] = {str(p.tp_keys[i]): p.comm_fixed[i] for i in range(p.n_tp)}
    d["num_experts"] = p.num_experts
    d["top_k"] = p.top_k
    d["deployment"] = {"tp": p.deploy_tp, "ep": p.deploy_ep, "dp": p.deploy_dp}
    return d


def write_profiles(ref: Reference) -> None:
    files = sorted(f for f in glob.glob(os.path.join(REF_DATA, "profiles", "*.json"))
                   if not f.endswith("platform.json"))
    profs = [profile_to_dict(ref.load_profile(f)) for f in files]
    gpu, k = ref.load_platform(os.path.join(REF_DATA, "profiles", "platform.json"))
    out = {
        "source": "reference proj/data/profiles via profile_from_json (json_io.hpp:70-105)",
        "platform": {
            "gpu": {"idle_watts": gpu.idle_watts, "min_cap_watts": gpu.min_cap_watts,
                    "max_cap_watts": gpu.max_cap_watts, "max_frequency": gpu.max_frequency},
            "system_power": {"alpha": k.alpha, "beta_watts": k.beta_watts},
        },
        "profiles": profs,
    }
    path = os.path.join(ROOT, "paper_2605_21427_b200", "data", "profiles.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    with open(os.path.join(REF_DATA, "grids", "full_grid.json")) as f:
        grid = json.load(f)
    with open(os.path.join(GOLD, "full_grid.json"), "w") as f:
        json.dump(grid, f)
        f.write("\n")


def fnv_bits(a: np.ndarray) -> int:
    h = 0xCBF29CE484222325
    for w in np.ascontiguousarray(a).view(np.uint64).tolist():
        h = ((h ^ w) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def gen_eval(ref: Reference) -> None:
    profs, gpu, _ = load_bundle()
    with open(os.path.join(GOLD, "full_grid.json")) as f:
        g = json.load(f)
    pts = workloads.grid_points(g["caps_w"], g["batches"], g["tps"], g["eps"], g["dps"])
    Ts, Ps, errs = [], [], []
    for p in profs:
        T, P, err = ref.eval(p, gpu, pts)
        Ts.append(T)
        Ps.append(P)
        errs.append(err)
    # off-grid points: caps inside/outside range, unknown tp, dp>1, batch 0
    rng = np.random.default_rng(7)
    n = 4000
    odd = np.zeros(n, POINT_DT)
    odd["cap_watts"] = rng.uniform(90.0, 410.0, n)
    odd["batch"] = rng.integers(0, 300, n)
    odd["tp"] = rng.choice([1, 2, 3, 4, 8], n)
    odd["ep"] = rng.integers(1, 9, n)
    odd["dp"] = rng.integers(1, 5, n)
    oT, oP, oerr = [], [], []
    for p in profs:
        T, P, err = ref.eval(p, gpu, odd)
        oT.append(T)
        oP.append(P)
        oerr.append(err)
    # cfg2 / cfg3 grids: bit digest + strided sample
    c2 = workloads.cfg2()
    T2, P2, e2 = ref.eval(c2["profile"], gpu, c2["points"])
    c3 = workloads.cfg3()
    T3, P3, e3 = ref.eval(c3["profile"], gpu, c3["points"])
    assert not e2.any() and not e3.any()
    np.savez_compressed(
        os.path.join(GOLD, "eval.npz"), full_points=pts, full_T=np.stack(Ts),
        full_P=np.stack(Ps), full_err=np.stack(errs), odd_points=odd, odd_T=np.stack(oT),
        odd_P=np.stack(oP), odd_err=np.stack(oerr),
        cfg2_T_sample=T2[::16], cfg2_P_sample=P2[::16],
        cfg2_digest=np.array([fnv_bits(T2), fnv_bits(P2)], np.uint64),
        cfg3_T_sample=T3[::16], cfg3_P_sample=P3[::16],
        cfg3_digest=np.array([fnv_bits(T3), fnv_bits(P3)], np.uint64))


def gen_select(ref: Reference) -> None:
    out = {}
    c1 = workloads.cfg1()
    T, P, _ = ref.eval(c1["profile"], c1["gpu"], c1["points"])
    tref = float(np.max(T * c1["points"]["dp"]))
    qs = [workloads.gen_queries(500, 11, tref, "qos"),
          workloads.gen_queries(500, 12, tref, "qos", budget=(900.0, 1900.0)),
          workloads.gen_queries(500, 13, tref, "mixed", budget=(700.0, 2100.0)),
          workloads.gen_queries(500, 14, tref, "budget", budget=(500.0, 1500.0))]
    q1 = np.concatenate(qs)
    i1, r1, rc = ref.select_analytic(c1["profile"], c1["gpu"], c1["points"], c1["coeffs"], q1)
    assert rc == 0
    out.update(cfg1_queries=q1, cfg1_idx=i1, cfg1_reason=r1)
    for name, cfg, specs in (
        ("cfg2", workloads.cfg2(), [("qos", None, 21, 200), ("qos", (600.0, 2000.0), 22, 200),
                                    ("mixed", (600.0, 2000.0), 23, 200)]),
        ("cfg3", workloads.cfg3(), [("mixed", (600.0, 2000.0), 2605, 300)]),
    ):
        T, P, _ = ref.eval(cfg["profile"], cfg["gpu"], cfg["points"])
        tref = float(np.max(T * cfg["points"]["dp"]))
        q = np.concatenate([workloads.gen_queries(n, s, tref, o, budget=b)
                            for (o, b, s, n) in specs])
        idx, rs, rc = ref.select_analytic(cfg["profile"], cfg["gpu"], cfg["points"],
                                          cfg["coeffs"], q)
        assert rc == 0
        out.update({f"{name}_queries": q, f"{name}_idx": idx, f"{name}_reason": rs,
                    f"{name}_tref": np.array([tref])})
    np.savez_compressed(os.path.join(GOLD, "select.npz"), **out)


def near_tie_tables(n_cases: int = 300, seed: int = 99):
    """Adversarial TableScorer cases: exact ties, 1e-10..1e-8 relative near-ties in
    t_hat, p_gpu and eff, duplicate points and duplicate (cap, batch) at different tp."""
    rng = np.random.default_rng(seed)
    cases = []
    for c in range(n_cases):
        n = int(rng.integers(2, 90))
        pts = np.zeros(n, POINT_DT)
        pts["cap_watts"] = rng.choice([150.0, 200.0, 250.0, 300.0, 400.0], n)
        pts["batch"] = rng.choice([1, 4, 8, 16, 32], n)
        pts["tp"] = rng.choice([1, 2, 4], n)
        pts["ep"] = 1
        pts["dp"] = rng.choice([1, 1, 1, 2], n)
        # unique points unless the case asks for duplicates (TableScorer first-match)
        if c % 7 != 0:
            key = (pts["cap_watts"] * 1000 + pts["batch"]) * 10 + pts["tp"]
            _, first = np.unique(key, return_index=True)
            pts = pts[np.sort(first)]
            n = len(pts)
        base_t = rng.uniform(100.0, 3000.0, max(1, n // 3))
        base_p = rng.uniform(60.0, 400.0, max(1, n // 3))
        T = base_t[rng.integers(0, len(base_t), n)].copy()
        P = base_p[rng.integers(0, len(base_p), n)].copy()
        mode = c % 5
        if mode == 1:  # t near-ties
            T *= 1.0 + rng.choice([0.0, 1e-10, 3e-10, 9e-10, 1.1e-9, 4e-9], n)
        elif mode == 2:  # p near-ties
            P *= 1.0 + rng.choice([0.0, -2e-10, 5e-10, 1e-9, 2e-9], n)
        elif mode == 3:  # chains of eff near-ties (non-transitive comparator)
            k = rng.uniform(0.5, 2.0)
            T = P * k * (1.0 + 0.9e-9 * rng.integers(0, 6, n))
        elif mode == 4:  # both
            T *= 1.0 + rng.choice([0.0, 5e-10, 1e-9], n)
            P *= 1.0 + rng.choice([0.0, 5e-10, 1e-9], n)
        tmax = float(np.max(T))
        nq = 24
        q = np.zeros(nq, QUERY_DT)
        q["throughput_tps"] = rng.uniform(0.05, 1.1, nq) * tmax
        q["bias"] = np.where(rng.uniform(size=nq) < 0.5, 1.0, rng.uniform(0.5, 2.0, nq))
        q["target_headroom"] = rng.choice([0.0, 0.05], nq)
        q["has_budget"] = rng.uniform(size=nq) < 0.6
        pn = 1.05 * 4 * P + 345.0
        q["power_budget_w"] = rng.uniform(0.9 * pn.min(), 1.1 * pn.max(), nq)
        q["budget_margin"] = rng.choice([0.0, 0.02], nq)
        q["objective"] = (rng.uniform(size=nq) < 0.3).astype(np.int32)
        cases.append((pts, T, P, q))
    return cases


def gen_tables(ref: Reference) -> None:
    _, _, coeffs = load_bundle()
    cases = near_tie_tables()
    pts, T, P, q, off, qoff, idx, rs = [], [], [], [], [0], [0], [], []
    for (p_, t_, pw_, q_) in cases:
        i, r, rc = ref.select_table(p_, t_, pw_, coeffs, q_)
        assert rc == 0, ref.last_error()
        pts.append(p_)
        T.append(t_)
        P.append(pw_)
        q.append(q_)
        off.append(off[-1] + len(p_))
        qoff.append(qoff[-1] + len(q_))
        idx.append(i)
        rs.append(r)
    np.savez_compressed(os.path.join(GOLD, "tables.npz"), points=np.concatenate(pts),
                        T=np.concatenate(T), P=np.concatenate(P), queries=np.concatenate(q),
                        off=np.array(off), qoff=np.array(qoff), idx=np.concatenate(idx),
                        reason=np.concatenate(rs))


def ladder(n, t_lo, t_hi):
    """test_controller.cpp:31-43"""
    pts = np.zeros(n, POINT_DT)
    T = np.zeros(n)
    P = np.zeros(n)
    for i in range(n):
        frac = 0.0 if n == 1 else i / (n - 1)
        thr = t_lo + (t_hi - t_lo) * frac
        pts[i] = (150.0 + i, 1 + i, 2, 1, 1)
        T[i] = thr
        P[i] = 40.0 + thr * thr / 800.0
    return pts, T, P


def gen_control(ref: Reference) -> None:
    """control_step sequences through the reference with a TableScorer ladder:
    lambda-biased plants (bias convergence), noise inside the dead-band, target
    steps, budget switches and stale telemetry."""
    from paper_2605_21427_b200.abi import default_ctrl_cfg
    from paper_2605_21427_b200.wattserve import make_targets
    _, _, coeffs = load_bundle()
    rng = np.random.default_rng(2024)
    recs = []
    seqs = []
    for s in range(60):
        n = [10, 30, 60, 160][s % 4]
        pts, T, P = ladder(n, 300.0, 2400.0)
        cfg = default_ctrl_cfg(target_headroom=[0.0, 0.05][s % 2],
                               budget_margin=[0.0, 0.02][(s // 2) % 2])
        st = CtrlState()
        st.bias = 1.0
        st.current = abi.Point(*pts[-1].tolist())
        lam = [0.7, 1.3, 1.0, 0.9][s % 4]
        tps = float(rng.uniform(700.0, 1500.0))
        obj = abi.OBJ_BUDGET if s % 5 == 4 else abi.OBJ_QOS
        budget = None
        now = 0.5
        cur_i = n - 1
        measured = lam * T[cur_i]
        for k in range(80):
            if k == 30:
                tps = float(rng.uniform(500.0, 2000.0))
            if k == 50 and s % 3 == 0:
                budget = float(1.05 * 4 * P[n // 2] + 345.0 + rng.uniform(-5.0, 5.0))
            tg = make_targets(tps, budget, 0.05, obj)
            t_s = now - (10.0 if (k % 17 == 16) else 0.0)  # occasional stale telemetry
            tel = Telemetry(t_s, measured)
            d, st2, rc = ref.control_step_table(pts, T, P, tel, now, tg, coeffs, st, cfg)
            assert rc == 0, ref.last_error()
            st = st2
            cur = st.current
            for i in range(n):
                if pts[i]["cap_watts"] == cur.cap_watts and pts[i]["batch"] == cur.batch:
                    cur_i = i
                    break
            measured = lam * T[cur_i] * (1.0 + float(rng.uniform(-0.03, 0.03)))
            recs.append((s, k, now, t_s, measured, tps, budget if budget is not None else np.nan,
                         obj, d.point.cap_watts, d.point.batch, d.applied, d.reason, st.bias,
                         st.integral, st.prev_error, st.has_prev_error, st.sustain_count,
                         st.current.cap_watts, st.current.batch))
            now += cfg.interval_s
        seqs.append((s, n, cfg.target_headroom, cfg.budget_margin, lam))
    dt = np.dtype([("seq", "i4"), ("k", "i4"), ("now", "f8"), ("t_s", "f8"), ("measured", "f8"),
                   ("tps", "f8"), ("budget", "f8"), ("objective", "i4"), ("d_cap", "f8"),
                   ("d_batch", "i4"), ("applied", "i4"), ("reason", "i4"), ("bias", "f8"),
                   ("integral", "f8"), ("prev_error", "f8"), ("has_prev", "i4"),
                   ("sustain", "i4"), ("cur_cap", "f8"), ("cur_batch", "i4")])
    sq = np.array(seqs, dtype=[("seq", "i4"), ("n", "i4"), ("headroom", "f8"), ("margin", "f8"),
                               ("lam", "f8")])
    np.savez_compressed(os.path.join(GOLD, "control.npz"), steps=np.array(recs, dtype=dt),
                        seqs=sq)


def gen_replay(ref: Reference) -> None:
    s = workloads.cfg4_setup()
    spec = workloads.replay_spec(96, n_steps=720, seed=515, n_log_traces=12)
    summ, logs = ref.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                            s["cfg"], spec)
    spec_q = workloads.replay_spec(32, n_steps=720, seed=516, objective_mode=0,
                                   n_log_traces=4)
    summ_q, logs_q = ref.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                                s["cfg"], spec_q)
    assert logs.dtype == STEPLOG_DT
    np.savez_compressed(os.path.join(GOLD, "replay.npz"), summ=summ, logs=logs, summ_q=summ_q,
                        logs_q=logs_q)


DECISION_SPECS = {  # name -> replay_spec kwargs of the decisions-CSV fixtures
    "mixed": dict(n_traces=24, n_steps=240, seed=2605, n_log_traces=12),
    "qos": dict(n_traces=8, n_steps=300, seed=77, objective_mode=0, n_log_traces=8),
    "dr": dict(n_traces=6, n_steps=200, seed=515, n_log_traces=6),
}


def write_scenarios() -> None:
    """The reference's bundled scenarios (proj/data/scenarios/*.json) with their budget
    traces resolved (budget_trace_csv, scenario_io.hpp:13-25, 46-49), as model-fit input
    for the queue-plant simulator: paper_2605_21427_b200/data/scenarios.json."""
    out = {}
    for f in sorted(glob.glob(os.path.join(REF_DATA, "scenarios", "*.json"))):
        with open(f) as fh:
            j = json.load(fh)
        trace = []
        if j.get("budget_trace_csv"):
            with open(os.path.join(os.path.dirname(f), j["budget_trace_csv"])) as fh:
                for line in fh:
                    line = line.strip()
                    if not line or not line[0].isdigit():
                        continue
                    t, w = line.split(",")
                    trace.append([float(t), float(w)])
        out[os.path.basename(f)[:-5]] = {"scenario": j, "trace": trace}
    with open(os.path.join(ROOT, "paper_2605_21427_b200", "data", "scenarios.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def gen_decisions(ref: Reference) -> None:
    """decisions_csv (metrics.hpp:145-157) produced by the reference's own writer over
    fluid-plant replays through the unmodified control_step, plus its fnv1a64."""
    s = workloads.cfg4_setup()
    out = {}
    for name, kw in DECISION_SPECS.items():
        spec = workloads.replay_spec(**kw)
        caps, batches = (workloads.dr_candidates() if name == "dr"
                         else (s["caps"], s["batches"]))
        csv, h = ref.replay_decisions_csv(s["profiles"], s["gpu"], s["coeffs"], caps, batches,
                                          s["cfg"], spec)
        out[name] = np.frombuffer(csv, np.uint8)
        out[name + "_fnv"] = np.array([h], np.uint64)
    np.savez_compressed(os.path.join(GOLD, "decisions.npz"), **out)


def forest_points(n, seed):
    rng = np.random.default_rng(seed)
    pts = np.zeros(n, POINT_DT)
    pts["cap_watts"] = np.where(rng.uniform(size=n) < 0.5, rng.uniform(100.0, 400.0, n),
                                rng.choice([150.0, 200.0, 250.0, 300.0, 350.0, 400.0], n))
    pts["batch"] = np.where(rng.uniform(size=n) < 0.5, rng.integers(1, 257, n),
                            rng.choice([1, 4, 8, 16, 32, 64], n))
    pts["tp"] = rng.choice([1, 2, 4, 8], n)
    pts["ep"] = rng.choice([1, 4, 8], n)
    pts["dp"] = rng.choice([1, 2, 3], n)
    return pts


def gen_forest(ref: Reference) -> None:
    """A small PredictorBundle (20 trees, depth 10) trained by the reference's own
    pipeline, shipped as model-fit input, plus the reference's predictions and
    predictor_scorer selections on it."""
    from oracle.oracle import ref_bundle_predict, ref_select_forest, ref_train_bundle
    from paper_2605_21427_b200.forest import Bundle
    profs, gpu, coeffs = load_bundle()
    path = "/tmp/pals_bundle_small.json"
    ref_train_bundle(ref, profs, gpu, coeffs, path, n_trees=20, max_depth=10, min_leaf=2,
                     seed=2605)
    b = Bundle.load_json(path)
    b.save_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data", "predictor_small.npz"))
    pts = forest_points(3000, 31)
    out = {"points": pts}
    for mid in ("llama2-7b-like", "mixtral-8x7b-like", "olmoe-like"):
        T, P, E = ref_bundle_predict(ref, path, mid, pts)
        out[f"{mid}_T"], out[f"{mid}_P"], out[f"{mid}_E"] = T, P, E
    # predictor_scorer selections over the cfg1 candidate grid of mixtral
    c1 = workloads.cfg1()
    mp = [p for p in profs if p.name.decode() == "mixtral-8x7b-like"][0]
    cands = workloads.grid_points(c1["caps"], c1["batches"], [mp.deploy_tp], [mp.deploy_ep],
                                  [mp.deploy_dp])
    T, _, _ = ref_bundle_predict(ref, path, "mixtral-8x7b-like", cands)
    q = np.concatenate([workloads.gen_queries(300, 41, float(T.max()), "qos"),
                        workloads.gen_queries(300, 42, float(T.max()), "mixed",
                                              budget=(800.0, 2000.0))])
    idx, rs = ref_select_forest(ref, path, "mixtral-8x7b-like", cands, coeffs, q)
    out.update(sel_points=cands, sel_queries=q, sel_idx=idx, sel_reason=rs)
    np.savez_compressed(os.path.join(GOLD, "forest.npz"), **out)


def gen_default_bundle(ref: Reference) -> None:
    """The PredictorBundle at the reference's default hyper-parameters (100 trees per
    forest, depth 14, min leaf 2: forest.hpp:72) trained by its own pipeline (run_sweep +
    train_bundle), shipped as model-fit input for the forest bench leg:
    paper_2605_21427_b200/data/predictor_default.npz."""
    import tempfile
    from oracle.oracle import ref_train_bundle
    from paper_2605_21427_b200.forest import Bundle
    profs, gpu, coeffs = load_bundle()
    path = os.path.join(tempfile.mkdtemp(), "bundle.json")
    ref_train_bundle(ref, profs, gpu, coeffs, path, n_trees=100, max_depth=14)
    Bundle.load_json(path).save_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data",
                                                 "predictor_default.npz"))


def main():
    os.makedirs(GOLD, exist_ok=True)
    ref = Reference()
    if len(sys.argv) > 1:  # regenerate only the named fixtures, e.g. "decisions"
        for name in sys.argv[1:]:
            globals()["gen_" + name](ref)
        return
    write_profiles(ref)
    write_scenarios()
    gen_eval(ref)
    gen_select(ref)
    gen_tables(ref)
    gen_control(ref)
    gen_replay(ref)
    gen_forest(ref)
    gen_decisions(ref)
    print("fixtures written to", GOLD)


if __name__ == "__main__":
    main()
