"""The N>1 path on CPU: world_size-2 gloo processes shard queries and replay
traces by contiguous global index, decide them independently with the C
oracle (standing in for each rank's GPU), and gather the results to rank 0,
which must equal the single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_21427_b200.shard import shard_range


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 10_000, 1_000_003):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0
            for (a, c), (b, _) in zip(spans, spans[1:]):
                assert a + c == b
            assert spans[-1][0] + spans[-1][1] == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2605_21427_b200 import workloads
    from paper_2605_21427_b200.shard import gather_to_rank0

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    # select: cfg1 grid, 403 queries sharded
    c1 = workloads.cfg1()
    T, P, _ = orc.eval(c1["profile"], c1["gpu"], c1["points"])
    nq = 403
    first, cnt = shard_range(nq, rank, world)
    q = workloads.gen_queries(cnt, 5, float(T.max()), "mixed", budget=(900.0, 1900.0),
                              first=first)
    idx, rs, rc = orc.select(c1["points"], T, P, c1["coeffs"], q)
    assert rc == 0
    packed = torch.from_numpy((idx.astype(np.int64) << 8) | rs.astype(np.int64))
    all_sel = gather_to_rank0(packed, nq, rank, world)
    # replay: 21 traces sharded
    s = workloads.cfg4_setup()
    nt = 21
    first, cnt = shard_range(nt, rank, world)
    spec = workloads.replay_spec(cnt, n_steps=300, seed=8, first=first)
    summ, _ = orc.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                         s["cfg"], spec)
    dig = torch.from_numpy(summ["digest"].view(np.int64).copy())
    all_dig = gather_to_rank0(dig, nt, rank, world)
    if rank == 0:
        np.savez(out_path, sel=all_sel.numpy(), dig=all_dig.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather(tmp_path, oracle):
    from paper_2605_21427_b200 import workloads
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    # single-process reference run
    c1 = workloads.cfg1()
    T, P, _ = oracle.eval(c1["profile"], c1["gpu"], c1["points"])
    q = workloads.gen_queries(403, 5, float(T.max()), "mixed", budget=(900.0, 1900.0))
    idx, rs, _ = oracle.select(c1["points"], T, P, c1["coeffs"], q)
    assert np.array_equal(got["sel"], (idx.astype(np.int64) << 8) | rs)
    s = workloads.cfg4_setup()
    summ, _ = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                            s["cfg"], workloads.replay_spec(21, n_steps=300, seed=8))
    assert np.array_equal(got["dig"], summ["digest"].view(np.int64))
