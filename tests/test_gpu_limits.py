"""Boundary shapes of the C ABI (include/sw_plan.h limits) on the GPU against the oracle:
the maximum numbers of scenes, digits, choices per digit, pools and queries, a one-plan
space, and every limit + 1 rejected with SW_EINVAL before any device work.

Expected values come only from oracle/ (live).  Integer results: exact equality."""
import random

import pytest

from swgen import INF
from swgen.generator import Query
from tests.conftest import cuda_available
from tests.helpers import make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sw():
    if not cuda_available():
        pytest.skip("no CUDA device")
    import paper_2603_05800_b200 as m
    m.lib()
    return m


def _problem(rng, S, first, radix, gpus, t_max=20_000_000):
    dur = [rng.randint(1, 60_000) * 1000 for _ in range(S)]
    llm = [rng.randint(0, 8_000_000) for _ in range(S)]
    tts = [rng.randint(0, 2_000_000) for _ in range(S)]
    choices, va = [], []
    for b, r in enumerate(radix):
        for _ in range(r):
            p = rng.randrange(len(gpus))
            choices.append((rng.randrange(4), rng.randint(1, gpus[p]), p))
        for _ in range(first[b], first[b + 1]):
            va.extend(rng.randint(1, t_max) for _ in range(r))
    price = [rng.choice([180250, 539500, 565250, 106500]) for _ in gpus]
    return make_problem(dur, llm, tts, gpus, price, radix, first, choices, va,
                        overhead_us=rng.randint(0, 2_000_000), fixed_cost_mc=rng.randint(0, 5000),
                        billing=rng.randrange(2), objective=rng.randrange(2), heads=0)


def _queries(rng, n):
    qs = [Query(INF, INF, INF), Query(0, 0, 0)]
    while len(qs) < n:
        qs.append(Query(rng.randint(0, 10**9), rng.randint(0, 10**9), rng.randint(0, 10**7)))
    return qs


def _full_parity(sw, orc, pb, qs):
    n = orc.n
    with sw.Plan(pb) as plan:
        assert plan.n == n
        plan.eval(0, n)
        got = plan.copy_records(0, n)
        exp = orc.records(0, n)
        for j in range(n):
            assert tuple(got[j].astuple()) == tuple(exp[j].astuple()), "record %d" % j
        w, f, d = orc.sweep(0, n, qs)
        sels = plan.select_batch(qs)
        for s, (st, idx, rec) in zip(sels, w):
            assert s.status == {0: 0, 1: 1, -1: 3}[st]
            if st >= 0:
                assert s.index == idx and tuple(s.rec) == rec.astuple()
        assert plan.pareto() == f
        assert plan.digest() == d


def test_max_scenes_digits_pools_queries(sw, oracle_mod):
    """64 scenes in 16 digits (SW_MAX_SCENES, SW_MAX_DIGITS) over 4 pools (SW_MAX_POOLS)
    with 8 queries (SW_MAX_QUERIES): 2^16 plans, every record, winners, front, digest."""
    rng = random.Random(71)
    S, B = 64, 16
    first = [4 * b for b in range(B)] + [S]
    pb = _problem(rng, S, first, [2] * B, [8, 4, 2, 1])
    qs = _queries(rng, 8)
    _full_parity(sw, oracle_mod.Oracle(pb), pb, qs)


def test_max_choices_per_digit(sw, oracle_mod):
    """One digit with 64 choices (SW_MAX_CHOICES) next to small ones, pools of up to 8 GPUs."""
    rng = random.Random(72)
    pb = _problem(rng, 6, [0, 1, 2, 6], [3, 64, 5], [8, 8, 3])
    _full_parity(sw, oracle_mod.Oracle(pb), pb, _queries(rng, 4))


def test_single_plan_space(sw, oracle_mod):
    """Every radix 1: N = 1 (one row, one tile of padding) -- winners, front, digest."""
    rng = random.Random(73)
    pb = _problem(rng, 5, [0, 2, 5], [1, 1], [4, 2])
    orc = oracle_mod.Oracle(pb)
    assert orc.n == 1
    _full_parity(sw, orc, pb, _queries(rng, 3))


def test_limits_plus_one_rejected(sw):
    """One beyond each limit fails at create with SW_EINVAL (host validation)."""
    rng = random.Random(74)
    # 65 scenes
    S = 65
    first = [5 * b for b in range(13)] + [S]
    bad = _problem(rng, S, first, [2] * 13, [2])
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(bad)
    assert ei.value.status == sw.SW_EINVAL
    # 17 digits
    S = 17
    bad = _problem(rng, S, list(range(S + 1)), [2] * S, [2])
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(bad)
    assert ei.value.status == sw.SW_EINVAL
    # 65 choices in a digit
    bad = _problem(rng, 3, [0, 1, 3], [65, 2], [2])
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(bad)
    assert ei.value.status == sw.SW_EINVAL
    # 5 pools
    bad = _problem(rng, 3, [0, 1, 3], [2, 2], [1, 1, 1, 1, 1])
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(bad)
    assert ei.value.status == sw.SW_EINVAL
    # 9 queries in one C call (the binding itself batches by SW_MAX_QUERIES)
    from paper_2603_05800_b200 import _native as nat
    pb = _problem(rng, 3, [0, 1, 3], [2, 2], [2])
    with sw.Plan(pb) as plan:
        plan.eval(0, plan.n)
        qs = _queries(rng, 9)
        arr = (nat.sw_query * 9)(*[nat.sw_query(q.slo_startup_us, q.slo_stall_us, q.budget_mc) for q in qs])
        out = (nat.sw_selection * 9)()
        assert nat.lib().sw_plan_select_batch(plan.h, 9, arr, out) == sw.SW_EINVAL


def test_empty_ranges(sw, oracle_mod):
    """eval of an empty range is a no-op; select with nothing evaluated is SW_EMPTY; a later
    eval of the whole space then matches the oracle."""
    rng = random.Random(75)
    pb = _problem(rng, 4, [0, 1, 2, 3, 4], [3, 2, 4, 2], [4, 2])
    orc = oracle_mod.Oracle(pb)
    qs = _queries(rng, 3)
    with sw.Plan(pb) as plan:
        plan.eval(5, 5)
        assert all(s.status == sw.SW_EMPTY for s in plan.select_batch(qs))
        plan.reset()
        plan.eval(0, plan.n)
        w, f, d = orc.sweep(0, orc.n, qs)
        for s, (st, idx, rec) in zip(plan.select_batch(qs), w):
            assert s.index == idx and tuple(s.rec) == rec.astuple()
        assert plan.pareto() == f
