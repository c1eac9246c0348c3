"""GPU parity with per-pool ready offsets (model load + warm-up; SURVEY §8(f)
row 3, reading R31) against the CPU oracle: records, winners, fronts, digests, details,
through the record path and the fused stream path.  Expected values come only from
oracle/ (live).  Integer results: exact equality."""
import random

import pytest

from swgen import make_config, INF
from swgen.generator import Query
from tests.helpers import random_problem
from tests.test_gpu_parity import _check_winners, _records_equal, sw  # noqa: F401 (fixture)

pytestmark = pytest.mark.gpu


def _exp(w):
    return [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]


@pytest.mark.parametrize("seed", range(10))
def test_random_problems_with_offsets(sw, oracle_mod, seed):  # noqa: F811
    rng = random.Random(3100 + seed)
    pb = random_problem(rng, max_scenes=7, max_pools=4, max_choices=5,
                        one_scene_digits=rng.random() < 0.5)
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
            assert list(sel.pool_end_us[:len(pb.gpus)]) == list(pend) and sel.makespan_us == mk
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(0, n, qs), _exp(w))
        assert plan.pareto() == f


def test_c3w_subrange(sw, oracle_mod):  # noqa: F811
    """C3 with a cold H100 pool (ready at 110 s): a ragged 3M sub-range through eval +
    select + front + digest and through the stream path; sampled records."""
    pb = make_config("C3w")
    b, e = 40_000_003, 43_000_017
    orc = oracle_mod.Oracle(pb)
    w, f, d = orc.sweep(b, e, pb.queries)
    with sw.Plan(pb, record_capacity=e - b + 10**6) as plan:
        plan.eval(b, e)
        _check_winners(plan.select_batch(pb.queries), _exp(w))
        assert plan.pareto() == f
        assert plan.digest() == d
        rng = random.Random(7)
        for _ in range(20):
            x = rng.randrange(b, e - 256)
            _records_equal(plan, orc, x, x + 256)
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(b, e, pb.queries), _exp(w))
        assert plan.pareto() == f
