"""K2 — the tree-ensemble predictor (PredictorBundle::predict, forest.hpp:227-235).

CPU: the C restatement is pinned against the reference's predictions on the
committed bundle (trained by the reference's own run_sweep + train_bundle) and,
where the reference build exists, against a freshly trained default bundle.
GPU: the cell-table path and the literal tree walk both reproduce the
reference bit for bit; predictor_scorer selections and a forest-scored
controller replay match.
"""
import os

import numpy as np
import pytest

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.forest import Bundle
from tests.helpers import bits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUNDLE = os.path.join(ROOT, "paper_2605_21427_b200", "data", "predictor_small.npz")
MODELS = ("llama2-7b-like", "mixtral-8x7b-like", "olmoe-like")


@pytest.fixture(scope="module")
def small_bundle():
    return Bundle.load_npz(BUNDLE)


def test_bundle_fixture_shape(small_bundle):
    b = small_bundle
    assert b.throughput.n_trees == 20 and b.power.n_trees == 20
    assert len(b.model_ids) == 8 and b.model_ids == sorted(b.model_ids)
    assert b.hyperparams == {"n_trees": 20, "max_depth": 10, "min_leaf": 2}


def test_oracle_forest_matches_reference_fixture(oracle, small_bundle, gold):
    from oracle.oracle import oracle_forest_predict
    g = gold("forest")
    for mid in MODELS:
        T, P, E = oracle_forest_predict(oracle, small_bundle, mid, g["points"])
        assert np.array_equal(bits(T), bits(g[f"{mid}_T"]))
        assert np.array_equal(bits(P), bits(g[f"{mid}_P"]))
        assert np.array_equal(bits(E), bits(g[f"{mid}_E"]))


def test_oracle_forest_select_matches_reference(oracle, small_bundle, gold, bundle):
    from oracle.oracle import oracle_forest_predict
    _, _, coeffs = bundle
    g = gold("forest")
    T, P, _ = oracle_forest_predict(oracle, small_bundle, "mixtral-8x7b-like", g["sel_points"])
    idx, rs, rc = oracle.select(g["sel_points"], T, P, coeffs, g["sel_queries"])
    assert rc == 0
    assert np.array_equal(idx, g["sel_idx"]) and np.array_equal(rs, g["sel_reason"])


def test_oracle_vs_reference_default_bundle(oracle, reference, bundle, tmp_path):
    """The reference's default hyper-parameters (100 trees, depth 14)."""
    from oracle.gen_golden import forest_points
    from oracle.oracle import oracle_forest_predict, ref_bundle_predict, ref_train_bundle
    profs, gpu, coeffs = bundle
    path = str(tmp_path / "bundle.json")
    ref_train_bundle(reference, profs, gpu, coeffs, path, n_trees=100, max_depth=14)
    b = Bundle.load_json(path)
    pts = forest_points(400, 77)
    for mid in MODELS:
        a = oracle_forest_predict(oracle, b, mid, pts)
        r = ref_bundle_predict(reference, path, mid, pts)
        for x, y in zip(a, r):
            assert np.array_equal(bits(x), bits(y))


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("direct", [False, True])
def test_gpu_forest_eval_bit_exact(ctx, small_bundle, gold, direct):
    from paper_2605_21427_b200.forest import make_forest_model
    from paper_2605_21427_b200.wattserve import Grid, eval_grid
    g = gold("forest")
    for mid in MODELS:
        m = make_forest_model(ctx, small_bundle, mid)
        assert ctx.lib.pals_model_forest_cells(m.h) > 0
        ctx.lib.pals_model_forest_set_direct(m.h, int(direct))
        T, P = eval_grid(m, Grid(ctx, g["points"]))
        assert np.array_equal(bits(T), bits(g[f"{mid}_T"]))
        assert np.array_equal(bits(P), bits(g[f"{mid}_P"]))


@pytest.mark.gpu
def test_gpu_forest_select_matches_reference(ctx, small_bundle, gold, bundle):
    from paper_2605_21427_b200.forest import make_forest_model
    from paper_2605_21427_b200.wattserve import Grid, Plan
    _, _, coeffs = bundle
    g = gold("forest")
    m = make_forest_model(ctx, small_bundle, "mixtral-8x7b-like")
    plan = Plan(m, Grid(ctx, g["sel_points"]), coeffs)
    idx, rs = plan.select(g["sel_queries"])
    assert np.array_equal(idx, g["sel_idx"]) and np.array_equal(rs, g["sel_reason"])


@pytest.mark.gpu
def test_gpu_forest_default_bundle_vs_reference(ctx, reference, bundle, tmp_path):
    """Default hyper-parameters (100 trees, depth 14) trained by the reference on the box."""
    from oracle.gen_golden import forest_points
    from oracle.oracle import ref_bundle_predict, ref_train_bundle
    from paper_2605_21427_b200.forest import make_forest_model
    from paper_2605_21427_b200.wattserve import Grid, eval_grid
    profs, gpu, coeffs = bundle
    path = str(tmp_path / "bundle.json")
    ref_train_bundle(reference, profs, gpu, coeffs, path, n_trees=100, max_depth=14)
    b = Bundle.load_json(path)
    pts = forest_points(20000, 78)
    for mid in MODELS:
        m = make_forest_model(ctx, b, mid)
        T, P = eval_grid(m, Grid(ctx, pts))
        rT, rP, _ = ref_bundle_predict(reference, path, mid, pts)
        assert np.array_equal(bits(T), bits(rT)) and np.array_equal(bits(P), bits(rP))


@pytest.mark.gpu
def test_gpu_forest_control_step_and_replay(ctx, oracle, small_bundle, bundle):
    """predictor_scorer drives the controller (the sim's Joint policy, sim.hpp:277-281):
    batched replay with forest scorers against the C oracle fed the same scores."""
    from oracle.oracle import oracle_forest_predict
    from paper_2605_21427_b200.forest import make_forest_model
    from paper_2605_21427_b200.wattserve import replay
    s = workloads.cfg4_setup()
    models, sT, sP = [], [], []
    for p in s["profiles"]:
        mid = p.name.decode()
        models.append(make_forest_model(ctx, small_bundle, mid))
        cands = workloads.grid_points(s["caps"], s["batches"], [p.deploy_tp], [p.deploy_ep],
                                      [p.deploy_dp])
        T, P, _ = oracle_forest_predict(oracle, small_bundle, mid, cands)
        sT.append(T)
        sP.append(P)
    spec = workloads.replay_spec(256, n_steps=1200, seed=11, n_log_traces=16)
    summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    osumm, ologs = oracle.replay_scored(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                        s["batches"], s["cfg"], spec, np.stack(sT), np.stack(sP))
    assert np.array_equal(logs, ologs)
    assert np.array_equal(summ, osumm)


@pytest.mark.gpu
def test_gpu_predict_device_points(ctx, small_bundle, gold):
    """pals_predict_device: PredictorBundle::predict over device-resident point records."""
    import torch

    from paper_2605_21427_b200.forest import make_forest_model
    g = gold("forest")
    pts = np.ascontiguousarray(g["points"])
    d_pts = torch.from_numpy(pts.view(np.uint8).copy()).cuda()
    for mid in MODELS:
        m = make_forest_model(ctx, small_bundle, mid)
        T = torch.empty(len(pts), dtype=torch.float64, device="cuda")
        P = torch.empty(len(pts), dtype=torch.float64, device="cuda")
        assert ctx.lib.pals_predict_device(ctx.h, m.h, d_pts.data_ptr(), len(pts), T.data_ptr(),
                                           P.data_ptr()) == 0
        ctx.sync()
        assert np.array_equal(bits(T.cpu().numpy()), bits(g[f"{mid}_T"]))
        assert np.array_equal(bits(P.cpu().numpy()), bits(g[f"{mid}_P"]))
