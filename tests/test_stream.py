"""GPU parity of the fused streaming path (sw_plan_stream) against
the CPU oracle: winners and the exact Pareto front of a range, with NO records stored.

Expected values come only from oracle/ (live, or tests/golden/ written by
tools/gen_golden.py from oracle/).  Integer results: exact equality.
"""
import random

import pytest

from swgen import make_config, INF
from swgen.generator import Query
from tests.conftest import cuda_available
from tests.helpers import random_problem
from tests.test_gpu_parity import _check_winners, _golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sw():
    if not cuda_available():
        pytest.skip("no CUDA device")
    import paper_2603_05800_b200 as m
    m.lib()
    return m


def _exp(w):
    return [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]


def _queries(rng):
    return [Query(INF, INF, INF),
            Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**6)),
            Query(INF, 0, INF),
            Query(0, 0, 0),                          # nothing feasible: closest tier
            Query(INF, INF, rng.randint(0, 10**6))]  # budget only (front-answerable)


@pytest.mark.parametrize("seed", range(12))
def test_stream_random_problems(sw, oracle_mod, seed):
    """Random small problems (both objectives, both billings, blocks of several scenes):
    stream == oracle sweep, winners and front."""
    rng = random.Random(500 + seed)
    pb = random_problem(rng, max_scenes=7, max_pools=3, max_choices=6,
                        one_scene_digits=rng.random() < 0.5)
    pb.queries = _queries(rng)
    orc = oracle_mod.Oracle(pb)
    with sw.Plan(pb, record_capacity=1024) as plan:
        n = plan.n
        w, f, _ = orc.sweep(0, n, pb.queries)
        _check_winners(plan.stream(0, n, pb.queries), _exp(w))
        assert plan.pareto() == f


@pytest.mark.parametrize("cfg", ["C1", "C2", "C2x", "C3", "C5"])
def test_stream_full_space(sw, cfg):
    """The configs' full spaces (C2: 4.3e8 plans; C5: 1.2e10 plans, whole-space golden) with
    a record capacity of 1024: the paper-shaped queries' winners and the front equal the
    oracle's (golden); C2x runs the paper's COST_X_TTFF objective."""
    pb = make_config(cfg)
    g = _golden(cfg)
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(0, plan.n, pb.queries), g["winners"])
        assert plan.pareto() == [tuple(p) for p in g["front"]]


def test_stream_c5_subranges(sw):
    """C5 (1.2e10 plans, 3 pools, 60 scenes) on the oracle's pinned sub-ranges."""
    g = _golden("C5sub")
    pb = make_config("C5")
    for rg in g["ranges"]:
        with sw.Plan(pb, record_capacity=1024) as plan:
            _check_winners(plan.stream(rg["begin"], rg["end"], pb.queries), rg["winners"])
            assert plan.pareto() == [tuple(p) for p in rg["front"]]


def test_stream_ragged_and_split(sw, oracle_mod):
    """A ragged C3 sub-range streamed in two calls: the front accumulates, the per-call
    winners merge (sw_selection_merge) to the oracle's winners of the whole range."""
    pb = make_config("C3")
    b, m, e = 7_000_001, 8_123_457, 9_876_543
    orc = oracle_mod.Oracle(pb)
    w, f, _ = orc.sweep(b, e, pb.queries)
    with sw.Plan(pb, record_capacity=1024) as plan:
        s1 = plan.stream(b, m, pb.queries)
        s2 = plan.stream(m, e, pb.queries)
        merged = [sw.selection_merge(pb.objective, q, x, y) for q, x, y in zip(pb.queries, s1, s2)]
        _check_winners(merged, _exp(w))
        assert plan.pareto() == f
        plan.reset()
        plan.eval(0, 100)
        with pytest.raises(sw.SwError) as ei:  # records held: stream refuses
            plan.stream(200, 300, pb.queries)
        assert ei.value.status == sw.SW_ESTATE


def test_stream_matches_eval_select(sw):
    """Same handle type, two paths: stream == eval + select_batch + pareto (C3 prefix)."""
    pb = make_config("C3")
    n = 3_000_017
    with sw.Plan(pb, record_capacity=n) as p1, sw.Plan(pb, record_capacity=1024) as p2:
        p1.eval(0, n)
        a = p1.select_batch(pb.queries)
        fa = p1.pareto()
        b = p2.stream(0, n, pb.queries)
        assert [(x.status, x.index, tuple(x.rec), x.digit) for x in a] == \
               [(x.status, x.index, tuple(x.rec), x.digit) for x in b]
        assert p2.pareto() == fa
