"""GPU parity of the shared-pool fleet (reading R36) through the C ABI:
sw_shared_create + eval / select / Pareto / digest / detail vs the oracle's per-pool EDF
event simulation (or_shared_eval), bit-exact (integer records)."""
import json
import os
import random
import threading

import pytest

from swgen import make_shared, SharedFleet, INF
from swgen.generator import Query
from tests.conftest import cuda_available
from tests.helpers import random_problem

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sw():
    if not cuda_available():
        pytest.skip("no CUDA device")
    import paper_2603_05800_b200 as m
    m.lib()
    return m


def _golden(cfg):
    p = os.path.join(GOLDEN, "oracle_%s.json" % cfg)
    if not os.path.exists(p):
        pytest.skip("golden %s not generated" % cfg)
    return json.load(open(p))


def _check(sels, front, dg, g):
    for s, w in zip(sels, g["winners"]):
        assert s.status == {0: 0, 1: 1, -1: 3}[w["status"]], (s, w)
        assert s.index == w["index"] and tuple(s.rec) == tuple(w["rec"]), (s, w)
    assert front == [tuple(p) for p in g["front"]]
    assert dg == int(g["digest"])


@pytest.mark.parametrize("cfg", ["SF2", "SF3"])
def test_shared_full_space(sw, oracle_mod, cfg):
    """SF2 (two requests planned jointly, 1.7e7 joint plans) and SF3 (the 1/3 mix, a new
    relaxed request against real-time + batch background load): winners of every query,
    the exact front and the digest vs the oracle; sampled records element by element;
    per-request detail vs the oracle's simulation."""
    sf = make_shared(cfg)
    g = _golden(cfg)
    so = oracle_mod.SharedOracle(sf)
    with sw.SharedPlan(sf) as plan:
        assert plan.n == so.n
        plan.eval(0, plan.n)
        _check(plan.select_batch(sf.queries), plan.pareto(), plan.digest(), g)
        rng = random.Random(5)
        for _ in range(40):
            b = rng.randrange(plan.n - 64)
            got = plan.copy_records(b, 64)
            for j in range(64):
                f, _, _ = so.eval(b + j)
                assert tuple(got[j].astuple()) == f.astuple(), b + j
        for _ in range(20):
            i = rng.randrange(plan.n)
            per, ready = plan.shared_detail(i)
            f, oper, ordy = so.eval(i)
            assert [p[:5] for p in per] == [(r.ttff_us, r.stall_us, r.cost_mc, r.quality, r.stall_count)
                                            for r in oper]
            assert ready == ordy
            d, _ = plan.detail(i)
            assert tuple(d.rec) == f.astuple()


@pytest.mark.parametrize("seed", range(8))
def test_shared_random_fleets(sw, oracle_mod, seed):
    """Random small fleets (2-3 requests, 1-3 pools, random arrivals, SLOs incl. batch,
    some background requests, both billings): every record, winners, front, digest."""
    rng = random.Random(700 + seed)
    P = rng.randint(1, 3)
    reqs, fixed = [], []
    for r in range(rng.randint(2, 3)):
        pb = random_problem(rng, max_scenes=4, max_pools=1, max_choices=3, one_scene_digits=rng.random() < 0.6)
        pb.choices = [(l, min(k, 4), rng.randrange(P)) for (l, k, p) in pb.choices]
        reqs.append(pb)
        fixed.append(None if r < 2 or rng.random() < 0.5 else rng.randrange(pb.n_candidates))
    gpus = [rng.randint(4, 8) for _ in range(P)]
    price = [rng.choice([180250, 539500]) for _ in range(P)]
    billing = rng.randrange(2)
    for pb in reqs:
        pb.gpus, pb.price_mc, pb.billing = list(gpus), list(price), billing
    R = len(reqs)
    sf = SharedFleet("rnd", reqs, [rng.randint(0, 10**7) for _ in range(R)],
                     [rng.choice([INF, rng.randint(0, 10**8)]) for _ in range(R)],
                     [rng.choice([INF, rng.randint(0, 10**8)]) for _ in range(R)], fixed, gpus, price,
                     billing=billing, objective=rng.randrange(2))
    sf.queries = [Query(INF, INF, INF), Query(0, 0, INF), Query(rng.randint(0, 10**8), 0, rng.randint(0, 10**6))]
    so = oracle_mod.SharedOracle(sf)
    with sw.SharedPlan(sf) as plan:
        n = plan.n
        assert n == so.n
        cut = rng.randrange(n + 1)
        plan.eval(cut, n)
        plan.eval(0, cut)
        for b, e in ((0, cut), (cut, n)):
            if e > b:
                got = plan.copy_records(b, e - b)
                for j in range(e - b):
                    assert tuple(got[j].astuple()) == so.eval(b + j)[0].astuple(), b + j
        w, f, d = so.sweep(0, n, sf.queries)
        sels = plan.select_batch(sf.queries)
        for s, (st, idx, rec) in zip(sels, w):
            assert s.status == {0: 0, 1: 1, -1: 3}[st] and s.index == idx and tuple(s.rec) == rec.astuple()
        assert plan.pareto() == f
        assert plan.digest() == d


def test_shared_loopback_two_ranks(sw):
    """SF2 sharded over two emulated ranks (loopback communicator): same winners, front
    and digest as the oracle on both ranks."""
    sf = make_shared("SF2")
    g = _golden("SF2")
    comms = sw.comm_loopback_create(2)
    res, errs = [None, None], [None, None]

    def work(r):
        try:
            with sw.SharedPlan(sf, device=0, comm=comms[r], rank=r, nranks=2) as plan:
                plan.eval(0, plan.n)
                res[r] = (plan.select_batch(sf.queries), plan.pareto(), plan.digest())
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    for c in comms:
        sw.comm_destroy(c)
    assert not any(errs), errs
    for sels, front, dg in res:
        _check(sels, front, dg, g)


def test_shared_errors(sw):
    sf = make_shared("SF3")
    with sw.SharedPlan(sf) as plan:
        with pytest.raises(sw.SwError):
            plan.stream(0, plan.n, sf.queries)
        with pytest.raises(sw.SwError):
            plan.greedy()
    sf = make_shared("SF2")
    sf.fixed_index = [10**9, None]  # background plan out of range
    with pytest.raises(sw.SwError) as ei:
        sw.SharedPlan(sf)
    assert ei.value.status == sw.SW_EINVAL
