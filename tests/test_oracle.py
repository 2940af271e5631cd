"""The oracle is pinned before it is trusted: the plain-C restatement
(oracle/pals_oracle.c) must reproduce the reference's own known-answer tests
(tests/test_model.cpp, tests/test_controller.cpp) and, bit for bit, the
fixtures the unmodified reference produced (tests/golden, oracle/gen_golden.py).
CPU only."""
import glob
import os

import numpy as np
import pytest

from paper_2605_21427_b200 import abi, workloads
from paper_2605_21427_b200.abi import Coeffs, GpuSpec, Profile
from paper_2605_21427_b200.profiles import load_bundle, profile_from_dict
from tests.helpers import bits, run_control_sequences, table_cases, table_view

REF_PROFILES = "/root/reference/proj/data/profiles"


def kat_profile(**kw) -> Profile:
    """tests/test_model.cpp:12-31 test_profile()."""
    d = dict(name="test-moe", total_params_b=10.0, active_params_b=2.0, num_experts=8, top_k=2,
             compute_fixed=0.002, compute_per_seq=0.0008,
             comm_fixed_by_tp={"1": 0.0004, "2": 0.001, "4": 0.004}, comm_per_seq=0.0006,
             internode_factor=1.3, knee_watts=200.0, compute_power_base=120.0,
             compute_power_per_seq=6.0, comm_power=110.0, overlap=0.5,
             deployment={"tp": 2, "ep": 4, "dp": 1})
    d.update(kw)
    return profile_from_dict(d)


KAT_GPU = GpuSpec(40.0, 100.0, 400.0, 1.0)


def pt(cap, batch, tp=2, ep=4, dp=1):
    a = np.zeros(1, abi.POINT_DT)
    a[0] = (cap, batch, tp, ep, dp)
    return a


@pytest.mark.skipif(not os.path.isdir(REF_PROFILES), reason="reference data absent")
def test_profiles_json_matches_reference_loader(reference, bundle):
    profs, gpu, coeffs = bundle
    files = sorted(f for f in glob.glob(os.path.join(REF_PROFILES, "*.json"))
                   if not f.endswith("platform.json"))
    assert len(files) == len(profs) == 8
    for f, p in zip(files, profs):
        r = reference.load_profile(f)
        assert bytes(r) == bytes(p), f
    g, k = reference.load_platform(os.path.join(REF_PROFILES, "platform.json"))
    assert bytes(g) == bytes(gpu) and bytes(k) == bytes(coeffs)


def test_frequency_law_kats(oracle):
    """test_model.cpp:35-47"""
    p = kat_profile()
    assert oracle.effective_frequency(200.0, p, KAT_GPU) == (1.0, 0)
    assert oracle.effective_frequency(400.0, p, KAT_GPU) == (1.0, 0)
    assert oracle.effective_frequency(150.0, p, KAT_GPU)[0] == pytest.approx(0.5)
    assert oracle.effective_frequency(100.0, p, KAT_GPU)[0] == pytest.approx(0.4)
    assert oracle.effective_frequency(50.0, p, KAT_GPU)[1] == abi.PALS_ERANGE
    assert oracle.effective_frequency(450.0, p, KAT_GPU)[1] == abi.PALS_ERANGE


def test_model_kats(oracle):
    """test_model.cpp:61-107: overlap limits, unknown tp, the 20 tok/s throughput KAT."""
    p0 = kat_profile(overlap=0.0)
    T, P, e = oracle.eval(p0, KAT_GPU, pt(300.0, 16))
    assert e[0] == 0
    T, P, e = oracle.eval(kat_profile(), KAT_GPU, pt(300.0, 16, tp=3))
    assert e[0] == abi.PALS_ECONFIG
    p = kat_profile(overlap=0.0, compute_fixed=0.04, compute_per_seq=0.0,
                    comm_fixed_by_tp={"2": 0.01}, comm_per_seq=0.0, knee_watts=200.0)
    T, P, e = oracle.eval(p, KAT_GPU, pt(400.0, 1))
    assert T[0] == pytest.approx(20.0)
    # cap monotonicity (test_model.cpp:109-115)
    caps = [150.0, 200.0, 250.0, 300.0, 350.0, 400.0]
    pts = np.concatenate([pt(c, 32) for c in caps])
    T, _, _ = oracle.eval(kat_profile(), KAT_GPU, pts)
    assert np.all(np.diff(T) >= -1e-12)
    # power bounds (test_model.cpp:137-147)
    pts = np.concatenate([pt(c, b) for c in (150.0, 200.0, 300.0, 400.0) for b in (1, 8, 64)])
    _, P, _ = oracle.eval(kat_profile(), KAT_GPU, pts)
    assert np.all(P >= 40.0) and np.all(P <= pts["cap_watts"] + 1e-9)
    # invalid points: batch 0, degree 0, cap out of range
    for bad, code in ((pt(300.0, 0), abi.PALS_ECONFIG), (pt(300.0, 4, dp=0), abi.PALS_ECONFIG),
                      (pt(99.0, 4), abi.PALS_ERANGE)):
        assert oracle.eval(kat_profile(), KAT_GPU, bad)[2][0] == code


def test_system_power_kat():
    """test_model.cpp:149-161: alpha*sum + beta with 4 x 300 W = 1605 W (p_node formula)."""
    k = Coeffs(1.05, 345.0)
    assert 1.0 * (k.alpha * 4 * 300.0 + k.beta_watts) == pytest.approx(1605.0)


def test_eval_matches_reference_fixtures(oracle, bundle, gold):
    profs, gpu, _ = bundle
    g = gold("eval")
    for i, p in enumerate(profs):
        T, P, e = oracle.eval(p, gpu, g["full_points"])
        assert np.array_equal(e, g["full_err"][i])
        ok = e == 0
        assert np.array_equal(bits(T[ok]), bits(g["full_T"][i][ok]))
        assert np.array_equal(bits(P[ok]), bits(g["full_P"][i][ok]))
        T, P, e = oracle.eval(p, gpu, g["odd_points"])
        assert np.array_equal(e, g["odd_err"][i])
        ok = e == 0
        assert ok.sum() > 100
        assert np.array_equal(bits(T[ok]), bits(g["odd_T"][i][ok]))
        assert np.array_equal(bits(P[ok]), bits(g["odd_P"][i][ok]))
    from oracle.gen_golden import fnv_bits
    for name, cfg in (("cfg2", workloads.cfg2()), ("cfg3", workloads.cfg3())):
        T, P, e = oracle.eval(cfg["profile"], gpu, cfg["points"])
        assert not e.any()
        assert np.array_equal(bits(T[::16]), bits(g[f"{name}_T_sample"]))
        assert [fnv_bits(T), fnv_bits(P)] == g[f"{name}_digest"].tolist()


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_select_matches_reference_fixtures(oracle, bundle, gold, name):
    cfg = getattr(workloads, name)()
    g = gold("select")
    T, P, e = oracle.eval(cfg["profile"], cfg["gpu"], cfg["points"])
    q = g[f"{name}_queries"]
    if name != "cfg1":
        q = q[::4]  # the C oracle is O(n) per query; a quarter of the fixture keeps CPU time low
        want_i, want_r = g[f"{name}_idx"][::4], g[f"{name}_reason"][::4]
    else:
        want_i, want_r = g[f"{name}_idx"], g[f"{name}_reason"]
    idx, rs, rc = oracle.select(cfg["points"], T, P, cfg["coeffs"], q)
    assert rc == 0
    assert np.array_equal(idx, want_i)
    assert np.array_equal(rs, want_r)


def test_select_near_tie_tables_match_reference(oracle, bundle, gold):
    _, _, coeffs = bundle
    n = 0
    for pts, T, P, q, want_i, want_r in table_cases(gold):
        Ts, Ps, canon = table_view(pts, T, P)
        idx, rs, rc = oracle.select(pts, Ts, Ps, coeffs, q)
        assert rc == 0
        assert np.array_equal(canon[idx], want_i) and np.array_equal(rs, want_r)
        n += len(q)
    assert n >= 5000


def test_control_sequences_match_reference(oracle, bundle, gold):
    _, _, coeffs = bundle

    def step(pts, T, P, tel, now, tg, st, cfg):
        cur = np.zeros(1, abi.POINT_DT)
        cur[0] = (st.current.cap_watts, st.current.batch, st.current.tp, st.current.ep,
                  st.current.dp)
        i = np.nonzero((pts["cap_watts"] == cur["cap_watts"]) & (pts["batch"] == cur["batch"]))[0]
        d, st2, rc = oracle.control_step(pts, T, P, T[i[0]] if len(i) else 0.0, len(i) > 0, tel,
                                         now, tg, coeffs, st, cfg)
        assert rc == 0
        return d, st2

    assert run_control_sequences(gold, step) == []


def test_replay_matches_reference_fixtures(oracle, gold):
    s = workloads.cfg4_setup()
    g = gold("replay")
    spec = workloads.replay_spec(96, n_steps=720, seed=515, n_log_traces=12)
    summ, logs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                               s["cfg"], spec)
    assert np.array_equal(summ, g["summ"])
    assert np.array_equal(logs, g["logs"])
    spec = workloads.replay_spec(32, n_steps=720, seed=516, objective_mode=0, n_log_traces=4)
    summ, logs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                               s["cfg"], spec)
    assert np.array_equal(summ, g["summ_q"]) and np.array_equal(logs, g["logs_q"])
    # the fixture exercises re-selection, holds and both objectives
    assert g["summ"]["n_applied"].sum() > 50
    assert set(np.unique(g["logs"]["reason"]).tolist()) >= {0, 2, 3}


def test_oracle_vs_reference_live(oracle, reference, bundle):
    """Random points and random TableScorer queries straight against the reference build."""
    profs, gpu, coeffs = bundle
    rng = np.random.default_rng(1234)
    pts = np.zeros(3000, abi.POINT_DT)
    pts["cap_watts"] = rng.uniform(95.0, 405.0, 3000)
    pts["batch"] = rng.integers(0, 257, 3000)
    pts["tp"] = rng.choice([1, 2, 4], 3000)
    pts["ep"] = rng.integers(1, 9, 3000)
    pts["dp"] = rng.integers(1, 6, 3000)
    for p in profs:
        a = oracle.eval(p, gpu, pts)
        b = reference.eval(p, gpu, pts)
        assert np.array_equal(a[2], b[2])
        ok = a[2] == 0
        assert np.array_equal(bits(a[0][ok]), bits(b[0][ok]))
        assert np.array_equal(bits(a[1][ok]), bits(b[1][ok]))
    from oracle.gen_golden import near_tie_tables
    for pts, T, P, q in near_tie_tables(60, seed=4321):
        Ts, Ps, canon = table_view(pts, T, P)
        a = oracle.select(pts, Ts, Ps, coeffs, q)
        b = reference.select_table(pts, T, P, coeffs, q)
        assert np.array_equal(canon[a[0]], b[0]) and np.array_equal(a[1], b[1])


def test_replay_oracle_vs_reference_live(oracle, reference):
    s = workloads.cfg4_setup()
    spec = workloads.replay_spec(48, n_steps=900, seed=77, n_log_traces=6)
    a = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], s["cfg"],
                      spec)
    b = reference.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                         s["cfg"], spec)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_bundle_loads():
    profs, gpu, coeffs = load_bundle()
    assert [p.name.decode() for p in profs] == sorted(p.name.decode() for p in profs)
    assert gpu.min_cap_watts == 100.0 and coeffs.alpha == 1.05
