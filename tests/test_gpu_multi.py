"""The multi-GPU driver (pals_multi_*) on one B200 with several contexts (the N>1 path:
one worker thread, context and stream per listed device, contiguous shards, results
straight to host or gathered into device 0 with cudaMemcpyPeerAsync). Sharded results
must equal the one-context results byte for byte."""
import numpy as np
import pytest

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.multi import Multi
from paper_2605_21427_b200.wattserve import (AnalyticModel, ConfigError, Grid, Plan, replay,
                                             replay_traces)
from tests.test_traces import build_dr_traces

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[[0, 0], [0, 0, 0]], ids=["2ctx", "3ctx"])
def multi(request):
    m = Multi(request.param)
    yield m
    m.close()


@pytest.mark.parametrize("gather", [False, True])
def test_multi_select_equals_single(ctx, multi, gather):
    cfg = workloads.cfg3(20_000)
    plan = Plan(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, cfg["points"]),
                cfg["coeffs"])
    th, _, _ = plan.scores()
    q = workloads.gen_queries(20_001, 5, float(th.max()), "mixed", budget=(600.0, 2000.0))
    want_i, want_r = plan.select(q)
    multi.set_gather(gather)
    mid = multi.model_analytic(cfg["profile"], cfg["gpu"])
    got_i, got_r = multi.select(mid, cfg["points"], cfg["coeffs"], q)
    assert np.array_equal(got_i, want_i) and np.array_equal(got_r, want_r)
    # again with the cached per-rank plans, and fewer queries than ranks
    got_i, got_r = multi.select(mid, cfg["points"], cfg["coeffs"], q[:1])
    assert got_i[0] == want_i[0] and got_r[0] == want_r[0]
    assert (multi.last_ms() >= 0).all()
    multi.set_gather(False)


@pytest.mark.parametrize("gather", [False, True])
def test_multi_replay_equals_single(ctx, multi, gather):
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    spec = workloads.replay_spec(5001, n_steps=720, seed=41, n_log_traces=37)
    from paper_2605_21427_b200.wattserve import replay_with_details
    want, wlogs, wdet = replay_with_details(ctx, models, s["profiles"], s["gpu"], s["coeffs"],
                                            s["caps"], s["batches"], s["cfg"], spec)
    multi.set_gather(gather)
    ids = [multi.model_analytic(p, s["gpu"]) for p in s["profiles"]]
    got, logs, det = multi.replay(ids, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                  s["batches"], s["cfg"], spec, details=True)
    assert np.array_equal(got, want)
    assert np.array_equal(logs, wlogs) and np.array_equal(det, wdet)
    multi.set_gather(False)


def test_multi_replay_traces_equals_single(ctx, multi, reference):
    from tests.test_traces import ref_plant_constants
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    t_max, _, _ = ref_plant_constants(reference, s, s["caps"], s["batches"])
    tr, sig = build_dr_traces(s, t_max, n_per_model=5, n_steps=1500, seed=4)
    a = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], s["cfg"])
    want = replay_traces(ctx, models, *a, tr, sig, 1500, n_log_traces=7, details=True)
    ids = [multi.model_analytic(p, s["gpu"]) for p in s["profiles"]]
    got = multi.replay_traces(ids, *a, tr, sig, 1500, n_log_traces=7, details=True)
    for k in ("summaries", "logs", "details", "final_state", "final_plant"):
        assert np.array_equal(got[k], want[k]), k
    bad = tr.copy()
    bad["model"][len(tr) - 2] = 77  # lands in the last shard: reported by its global index
    with pytest.raises(ConfigError, match=f"trace {len(tr) - 2}: model index"):
        multi.replay_traces(ids, *a, bad, sig, 10)
