"""Pools of 9..32 GPUs (SURVEY §8(a) layout note, §8(b) "G_p <= 8 fast path, <= 32
generic"): the library's warp-per-candidate path (sw_wide.cuh) vs the oracle, bit-exact.
The paper's own setups use 16 x A100 and 64 x A100 servers."""
import json
import os
import random

import pytest

from swgen import make_config, INF
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


def _records_equal(plan, orc, b, e):
    got = plan.copy_records(b, e - b)
    exp = orc.records(b, e)
    for j in range(e - b):
        assert tuple(got[j].astuple()) == tuple(exp[j].astuple()), "record %d" % (b + j)


def _check(sels, w):
    for s, (st, idx, rec) in zip(sels, w):
        assert s.status == {0: 0, 1: 1, -1: 3}[st]
        if st >= 0:
            assert s.index == idx and tuple(s.rec) == rec.astuple()


@pytest.mark.parametrize("seed", range(10))
def test_wide_random(sw, oracle_mod, seed):
    """Random problems with pools of up to 32 GPUs and k up to 32 (both billings, both
    objectives, random blocks, ragged multi-call ranges): every record, winners, front,
    digest, winner details."""
    rng = random.Random(3000 + seed)
    pb = random_problem(rng, max_scenes=6, max_pools=3, max_g=32, max_choices=4,
                        one_scene_digits=rng.random() < 0.5)
    if max(pb.gpus) <= 8:
        pb.gpus[0] = rng.randint(9, 32)
    orc = oracle_mod.Oracle(pb)
    n = orc.n
    qs = [Query(INF, INF, INF), Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**6)),
          Query(0, 0, 0)]
    cuts = sorted({0, n} | {rng.randrange(n + 1) for _ in range(2)})
    with sw.Plan(pb) as plan:
        for a, b in zip(cuts[:-1], cuts[1:]):
            plan.eval(a, b)
        for a, b in zip(cuts[:-1], cuts[1:]):
            if b > a:
                _records_equal(plan, orc, a, b)
        w, f, d = orc.sweep(0, n, qs)
        sels = plan.select_batch(qs)
        _check(sels, w)
        assert plan.pareto() == f
        assert plan.digest() == d
        for s in sels:
            if s.status != sw.SW_EMPTY:
                sel, ready = plan.detail(s.index)
                rec, oready, pend, mk, te = orc.eval(s.index)
                assert tuple(sel.rec) == rec.astuple() and ready == oready
                assert sel.pool_end_us == pend and sel.makespan_us == mk and sel.ttff_eff_us == te


def test_wide_c2w_full_space(sw, oracle_mod):
    """C2 on a 16 x A100 pool: winners, exact front, digest over the full 12^8
    space vs the oracle golden; sampled records."""
    p = os.path.join(GOLDEN, "oracle_C2w.json")
    if not os.path.exists(p):
        pytest.skip("golden C2w not generated")
    g = json.load(open(p))
    pb = make_config("C2w")
    orc = oracle_mod.Oracle(pb)
    with sw.Plan(pb) as plan:
        plan.eval(0, plan.n)
        sels = plan.select_batch(pb.queries)
        for s, w in zip(sels, g["winners"]):
            assert s.status == {0: 0, 1: 1, -1: 3}[w["status"]]
            assert s.index == w["index"] and tuple(s.rec) == tuple(w["rec"])
        assert plan.pareto() == [tuple(x) for x in g["front"]]
        assert plan.digest() == int(g["digest"])
        rng = random.Random(17)
        for _ in range(30):
            b = rng.randrange(plan.n - 256)
            _records_equal(plan, orc, b, b + 256)


def test_wide_limits(sw):
    pb = make_config("C2w")
    with sw.Plan(pb, record_capacity=1 << 20) as plan:
        with pytest.raises(sw.SwError):
            plan.stream(0, 1000, pb.queries)  # the fused stream mode needs pools of <= 8 GPUs
        with pytest.raises(sw.SwError):
            plan.greedy()
    bad = make_config("C2w")
    bad.gpus = [33]
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(bad)
    assert ei.value.status == sw.SW_EINVAL
