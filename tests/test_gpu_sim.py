"""K6 queue-plant simulator vs the unmodified reference run_scenario (sim.hpp:482-485):
the three bundled scenarios x the five policies in ONE batched GPU call, every
telemetry / decision log entry, every per-node MetricsSummary, the arrival-stream
hashes, the RunSummary aggregates and the reference's CSV bytes."""
import os
import tempfile

import numpy as np
import pytest

from paper_2605_21427_b200.abi import POLICIES
from paper_2605_21427_b200.forest import Bundle, make_forest_model
from paper_2605_21427_b200.sim import (bundled_scenarios, decisions_csv, n_intervals,
                                       requests_csv, run_scenarios, telemetry_csv)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NODE_FIELDS = ["tokens_per_joule", "qos_violation_rate", "power_tracking_mae_w", "total_tokens",
               "total_energy_j", "mean_throughput_tps", "throughput_target_tps", "final_bias",
               "arrival_stream_hash", "n_requests", "n_completed", "n_applied"]
RES_FIELDS = ["tokens_per_joule", "qos_violation_rate", "power_tracking_mae_w", "total_tokens",
              "total_energy_j", "mean_throughput_tps", "cluster_tracking_mae_w",
              "sim_total_energy_j", "n_intervals"]


@pytest.fixture(scope="module")
def setup(ctx, bundle):
    profs, gpu, coeffs = bundle
    b = Bundle.load_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data",
                                     "predictor_small.npz"))
    path = os.path.join(tempfile.mkdtemp(), "bundle.json")
    b.to_json(path)
    preds = {p.name.decode(): make_forest_model(ctx, b, p.name.decode()) for p in profs}
    return profs, gpu, coeffs, preds, path


def _check(ours, ref, sc, tag):
    nres, res, tel, dec = ours
    rn, rr, rt, rd = ref
    n = n_intervals(sc)
    for f in NODE_FIELDS:
        assert np.array_equal(nres[f], rn[f]), (tag, f, nres[f], rn[f])
    for f in RES_FIELDS:
        assert res[f] == rr[f], (tag, f, res[f], rr[f])
    assert np.array_equal(tel[:, :n], rt), tag
    assert np.array_equal(dec[:, :n], rd), tag


def test_bundled_scenarios_all_policies(ctx, reference, setup):
    profs, gpu, coeffs, preds, path = setup
    scs, tags = [], []
    for name, sc in sorted(bundled_scenarios().items()):
        for pol in POLICIES:
            scs.append(dict(sc, policy=pol))
            tags.append(f"{name}/{pol}")
    nres, res, tel, dec, reqs = run_scenarios(ctx, scs, profs, gpu, coeffs, preds, logs=True,
                                              requests=True)
    o = 0
    for i, (sc, tag) in enumerate(zip(scs, tags)):
        k = len(sc["nodes"])
        ref = reference.run_scenario(sc, profs, gpu, coeffs, path, want_csv=True)
        ours = (nres[o:o + k], res[i], tel[o:o + k], dec[o:o + k])
        _check(ours, ref[:4], sc, tag)
        tcsv, dcsv, rcsv = ref[4]
        assert telemetry_csv(sc, tel[o:o + k]) == tcsv, tag
        assert decisions_csv(sc, tel[o:o + k], dec[o:o + k]) == dcsv, tag
        assert requests_csv(sc, reqs[o:o + k]) == rcsv, tag
        o += k


def test_seed_sweep_and_variants(ctx, reference, setup):
    """Other seeds, interval lengths, backlog / arrival rates, a dp=2 node, no predictor
    for the oracle, margins; static budgets below / above the draw."""
    profs, gpu, coeffs, preds, path = setup
    base = bundled_scenarios()
    rng = np.random.default_rng(5)
    scs = []
    for case in range(12):
        sc = dict(base[["single_node", "multinode_qos", "demand_response"][case % 3]])
        sc["seed"] = int(rng.integers(1, 1 << 40))
        sc["duration_s"] = float(rng.choice([60.0, 150.0, 300.0]))
        sc["policy"] = list(POLICIES)[case % 5]
        nodes = []
        for nd in sc["nodes"]:
            nd = dict(nd, arrival_rate_per_s=float(rng.uniform(0.0, 14.0)),
                      initial_backlog=int(rng.integers(0, 300)))
            if case % 4 == 1:
                nd["dp"] = 2
            nodes.append(nd)
        sc["nodes"] = nodes
        if case % 3 == 1:
            sc["cluster_budget_w"] = float(rng.uniform(1800.0, 6000.0))
        if case % 6 == 0:
            sc["interval_s"] = 0.25
        scs.append(sc)
    nres, res, tel, dec = run_scenarios(ctx, scs, profs, gpu, coeffs, preds, logs=True)
    o = 0
    for i, sc in enumerate(scs):
        k = len(sc["nodes"])
        try:
            ref = reference.run_scenario(sc, profs, gpu, coeffs, path)
        except RuntimeError:
            pytest.fail(f"reference rejected case {i}")
        _check((nres[o:o + k], res[i], tel[o:o + k], dec[o:o + k]), ref, sc, f"case{i}")
        o += k


def test_errors_follow_the_reference(ctx, reference, setup):
    """Invalid scenarios fail like run_scenario / summarize would (same exception kinds)."""
    from paper_2605_21427_b200._lib import ConfigError, DataError
    profs, gpu, coeffs, preds, path = setup
    base = bundled_scenarios()["single_node"]
    with pytest.raises(ConfigError, match="policy requires a trained predictor"):
        run_scenarios(ctx, [dict(base, policy="joint")], profs, gpu, coeffs, None)
    with pytest.raises(RuntimeError):  # the reference refuses it the same way
        reference.run_scenario(dict(base, policy="joint"), profs, gpu, coeffs, None)
    with pytest.raises(ConfigError, match="qos_fraction"):
        bad = dict(base, nodes=[dict(base["nodes"][0], qos_fraction=1.5)])
        run_scenarios(ctx, [bad], profs, gpu, coeffs, preds)
    with pytest.raises(DataError, match="empty telemetry log"):
        run_scenarios(ctx, [dict(base, duration_s=0.1)], profs, gpu, coeffs, preds)
    with pytest.raises(ConfigError, match="at most 32 nodes"):
        big = dict(base, nodes=[base["nodes"][0]] * 33)
        run_scenarios(ctx, [big], profs, gpu, coeffs, preds)
    # joint split of a cluster budget below the nodes' floors: allocate_budget throws
    mn = bundled_scenarios()["multinode_qos"]
    low = dict(mn, cluster_budget_w=100.0)
    with pytest.raises(ConfigError):
        run_scenarios(ctx, [low], profs, gpu, coeffs, preds)
    with pytest.raises(RuntimeError):
        reference.run_scenario(low, profs, gpu, coeffs, path)


def test_streamed_upload_matches_upload_first(ctx, setup):
    """The streamed arrival upload (k_sim launched after the first chunk of intervals) and
    the profiler mode (every chunk uploaded before the launch) give the same bytes."""
    profs, gpu, coeffs, preds, _ = setup
    scs = []
    for seed in range(4):
        for sc in bundled_scenarios().values():
            for pol in POLICIES:
                scs.append(dict(sc, policy=pol, seed=seed))
    a = run_scenarios(ctx, scs, profs, gpu, coeffs, preds, logs=True)
    ctx.set_sim_streaming(False)
    try:
        b = run_scenarios(ctx, scs, profs, gpu, coeffs, preds, logs=True)
    finally:
        ctx.set_sim_streaming(True)
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()
