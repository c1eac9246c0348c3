"""Spot VMs with over-provisioning by eviction risk (Table 3 Spot column
P:633-638; reading R32).

CPU part: the oracle pinned to SPEC's worked Spot cost, to the closed form of the
billed GPU count n = the fewest GPUs with n (1 - rho) >= G (boundaries worked out by hand
below), and to the invariant that a Spot risk changes only the bill.  GPU part: parity of
the CUDA path with the oracle (records, winners, fronts, digests, details, stream path) on
random problems with random risks and on a ragged sub-range of C3s.  Expected values come
only from oracle/ (live) or from the hand-worked numbers cited here."""
import random

import pytest

from swgen import make_config, INF
from swgen.generator import Query, GPU_CLASSES
from tests.helpers import make_problem, random_problem
from tests.test_gpu_parity import sw  # noqa: F401 (GPU fixture: skips without CUDA)

H100_SPOT_MC = 402_750  # Table 3: $32.22 per 8-GPU server-hour -> mc per GPU-hour


def _one_scene(gpus, price, span_us, k=None):
    """One scene on one pool, no fixed stages: the pool is busy (and billed) for span_us."""
    k = gpus if k is None else k
    return make_problem([1_000_000], [0], [0], [gpus], [price], [1], [0, 1], [(0, k, 0)],
                        [span_us], heads=0)


def test_spec_worked_spot_cost(oracle_mod):
    """4xH100 Spot for 1800 s -> $32.22 x (4/8) x 0.5 = $8.055 = 805,500 mc.
    With a 20% eviction risk the pool needs n with n x 0.8 >= 4 -> n = 5 GPUs:
    $32.22 x (5/8) x 0.5 = $10.06875 = 1,006,875 mc."""
    pb = _one_scene(4, H100_SPOT_MC, 1_800_000_000)
    assert GPU_CLASSES["H100"][2] == H100_SPOT_MC
    assert oracle_mod.Oracle(pb).eval(0)[0].cost_mc == 805_500
    pb.evict_risk_permille = [200]
    assert oracle_mod.Oracle(pb).eval(0)[0].cost_mc == 1_006_875


# (G, rho per mille) -> billed GPUs, worked by hand from n (1 - rho) >= G:
# 8 x 1000/900 = 8.89 -> 9; 8000/889 = 8.9989 -> 9; 8000/888 = 9.009 -> 10;
# 8 / 0.8 = 10 exactly -> 10; 8000/799 = 10.01 -> 11; 1 / 0.5 = 2; 1000/1 = 1000 at 999.
BILLED = [((8, 0), 8), ((8, 1), 9), ((8, 100), 9), ((8, 111), 9), ((8, 112), 10),
          ((8, 200), 10), ((8, 201), 11), ((1, 500), 2), ((3, 500), 6), ((2, 999), 2000),
          ((32, 50), 34)]


@pytest.mark.parametrize("g_rho,n", BILLED)
def test_billed_gpu_count(oracle_mod, g_rho, n):
    """Price 1000 mc per GPU-hour and a 1-hour span: the pool bill is exactly 1000 x n."""
    G, rho = g_rho
    pb = _one_scene(G, 1000, 3_600_000_000)
    pb.evict_risk_permille = [rho]
    rec = oracle_mod.Oracle(pb).eval(0)[0]
    assert rec.cost_mc == 1000 * n


def test_risk_changes_only_the_bill(oracle_mod):
    """Over-provisioned spares stand by: times, quality, stall counts and pools used are
    those of the risk-free plan; the bill never drops; a 50% risk on a single pool doubles
    its billed GPUs (closed form)."""
    rng = random.Random(3200)
    for _ in range(150):
        pb = random_problem(rng, max_scenes=5, max_pools=3)
        pb.billing = 0
        base = oracle_mod.Oracle(pb)
        pb.evict_risk_permille = [rng.choice([0, rng.randint(1, 999)]) for _ in pb.gpus]
        spot = oracle_mod.Oracle(pb)
        for i in {0, base.n - 1, rng.randrange(base.n)}:
            r0, ready0, pend0, mk0, te0 = base.eval(i)
            r1, ready1, pend1, mk1, te1 = spot.eval(i)
            assert (r1.ttff_us, r1.stall_us, r1.quality, r1.stall_count, r1.flags) == \
                   (r0.ttff_us, r0.stall_us, r0.quality, r0.stall_count, r0.flags)
            assert (ready1, pend1, mk1, te1) == (ready0, pend0, mk0, te0)
            assert r1.cost_mc >= r0.cost_mc
    for _ in range(100):
        G = rng.randint(1, 8)
        span = rng.randint(1, 10**10)
        price = rng.choice([106_500, 180_250, 402_750, 539_500])
        pb = _one_scene(G, price, span, k=rng.randint(1, G))
        pb.evict_risk_permille = [500]
        got = oracle_mod.Oracle(pb).eval(0)[0].cost_mc
        pb2 = _one_scene(2 * G, price, span, k=pb.choices[0][1])
        assert got == oracle_mod.Oracle(pb2).eval(0)[0].cost_mc


@pytest.fixture(scope="module")
def swlib():
    from paper_2603_05800_b200 import build
    build.build()
    import paper_2603_05800_b200 as m
    return m


def test_busy_billing_rejects_risk(swlib, oracle_mod):
    """BUSY billing has no idle spares to bill (R32): the oracle refuses, and the library
    returns SW_EINVAL on the host before any device call; so does rho >= 1000."""
    pb = _one_scene(4, H100_SPOT_MC, 1_000_000)
    pb.billing = 1
    pb.evict_risk_permille = [100]
    with pytest.raises(ValueError):
        oracle_mod.Oracle(pb)
    with pytest.raises(swlib.SwError) as ei:
        swlib.Plan(pb)
    assert ei.value.status == swlib.SW_EINVAL
    pb.billing = 0
    pb.evict_risk_permille = [1000]
    with pytest.raises(swlib.SwError) as ei:
        swlib.Plan(pb)
    assert ei.value.status == swlib.SW_EINVAL


def test_c3s_config():
    """C3s = C3 with the H100 pool on Table 3's Spot column and a 10% risk."""
    a, b = make_config("C3"), make_config("C3s")
    assert b.price_mc == [180_250, 402_750] and b.evict_risk_permille == [0, 100]
    assert (a.va_us, a.choices, a.gpus) == (b.va_us, b.choices, b.gpus)


# ---------------------------------------------------------------- GPU parity


def _exp(w):
    return [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_gpu_random_problems_with_risk(sw, oracle_mod, seed):  # noqa: F811
    from tests.test_gpu_parity import _check_winners, _records_equal
    rng = random.Random(3300 + seed)
    pb = random_problem(rng, max_scenes=7, max_pools=4, max_choices=5,
                        one_scene_digits=rng.random() < 0.5)
    pb.billing = 0
    pb.evict_risk_permille = [rng.choice([0, rng.randint(1, 999)]) for _ in pb.gpus]
    if rng.random() < 0.5:
        pb.pool_ready_us = [rng.choice([0, rng.randint(0, 300_000_000)]) for _ in pb.gpus]
    orc = oracle_mod.Oracle(pb)
    n = orc.n
    qs = [Query(INF, INF, INF), Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**6)),
          Query(0, 0, 0), Query(INF, INF, rng.randint(0, 10**6))]
    w, f, d = orc.sweep(0, n, qs)
    with sw.Plan(pb) as plan:
        plan.eval(0, n)
        _records_equal(plan, orc, 0, n)
        _check_winners(plan.select_batch(qs), _exp(w))
        assert plan.pareto() == f
        assert plan.digest() == d
        for i in {0, n - 1, rng.randrange(n)}:
            sel, ready = plan.detail(i)
            rec, ready_o, pend, mk, te = orc.eval(i)
            assert tuple(sel.rec) == rec.astuple() and list(ready) == list(ready_o)
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(0, n, qs), _exp(w))
        assert plan.pareto() == f


@pytest.mark.gpu
def test_gpu_c3s_subrange(sw, oracle_mod):  # noqa: F811
    """C3s: a ragged 3M sub-range through eval + select + front + digest and through the
    stream path; sampled records."""
    from tests.test_gpu_parity import _check_winners, _records_equal
    pb = make_config("C3s")
    b, e = 50_000_011, 53_000_029
    orc = oracle_mod.Oracle(pb)
    w, f, d = orc.sweep(b, e, pb.queries)
    with sw.Plan(pb, record_capacity=e - b + 10**6) as plan:
        plan.eval(b, e)
        _check_winners(plan.select_batch(pb.queries), _exp(w))
        assert plan.pareto() == f
        assert plan.digest() == d
        rng = random.Random(11)
        for _ in range(20):
            x = rng.randrange(b, e - 256)
            _records_equal(plan, orc, x, x + 256)
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(b, e, pb.queries), _exp(w))
        assert plan.pareto() == f
