"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Every value compared here comes from oracle/ (live, or tests/golden/ written by
tools/gen_golden.py which calls only oracle/).  Integer results: exact equality.
"""
import json
import os
import random

import pytest

from swgen import make_config, make_fleet, INF
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


def _rec(r):
    return tuple(r.astuple()) if hasattr(r, "astuple") else tuple(r)


def _check_winners(sels, gwin):
    for s, w in zip(sels, gwin):
        st = {0: 0, 1: 1, -1: 3}[w["status"]]
        assert s.status == st
        if st != 3:
            assert s.index == w["index"]
            assert tuple(s.rec) == tuple(w["rec"])


def _records_equal(plan, orc, b, e):
    got = plan.copy_records(b, e - b)
    exp = orc.records(b, e)
    for j in range(e - b):
        assert _rec(got[j]) == _rec(exp[j]), "record %d" % (b + j)


def test_c1_exhaustive(sw, oracle_mod):
    pb = make_config("C1")
    g = _golden("C1")
    orc = oracle_mod.Oracle(pb)
    with sw.Plan(pb) as plan:
        assert plan.n == 256
        plan.eval(0, 256)
        _records_equal(plan, orc, 0, 256)
        _check_winners(plan.select_batch(pb.queries), g["winners"])
        assert plan.pareto() == [tuple(p) for p in g["front"]]
        assert plan.digest() == int(g["digest"])
        assert plan.launch_count() > 0


@pytest.mark.parametrize("seed", range(12))
def test_random_problems_all_records(sw, oracle_mod, seed):
    """Random shapes (B = 1..6 digits, 1..4 pools, G <= 8, runtime k) incl. the padded
    B < 3 layouts; ragged multi-call ranges; records, winners, front, digest."""
    rng = random.Random(1000 + seed)
    pb = random_problem(rng, max_scenes=7, max_pools=4, max_choices=5,
                        one_scene_digits=rng.random() < 0.5)
    orc = oracle_mod.Oracle(pb)
    n = orc.n
    cuts = sorted({0, n} | {rng.randrange(n + 1) for _ in range(rng.randint(0, 3))})
    qs = [Query(INF, INF, INF), Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**6)),
          Query(0, 0, 0)]
    with sw.Plan(pb) as plan:
        for a, b in zip(cuts[:-1], cuts[1:]):
            plan.eval(a, b)
        for a, b in zip(cuts[:-1], cuts[1:]):
            if b > a:
                _records_equal(plan, orc, a, b)
        w, f, d = orc.sweep(0, n, qs)
        sels = plan.select_batch(qs)
        _check_winners(sels, [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w])
        assert plan.pareto() == f
        assert plan.digest() == d


def test_detail_matches_oracle(sw, oracle_mod):
    rng = random.Random(5)
    for cfg in ["C1", "C2", "C3", "C5"]:
        pb = make_config(cfg)
        orc = oracle_mod.Oracle(pb)
        with sw.Plan(pb, record_capacity=1) as plan:
            for _ in range(20):
                i = rng.randrange(orc.n)
                sel, ready = plan.detail(i)
                rec, oready, pend, mk, te = orc.eval(i)
                assert tuple(sel.rec) == rec.astuple()
                assert ready == oready
                assert sel.pool_end_us == pend
                assert sel.makespan_us == mk and sel.ttff_eff_us == te
                assert sel.digit == orc.decode(i)


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_space(sw, oracle_mod, cfg):
    """Full space at the bench's launch configuration: winners, front and digest vs the
    oracle's full sweep; 200 sampled runs of 512 records element by element."""
    pb = make_config(cfg)
    g = _golden(cfg)
    orc = oracle_mod.Oracle(pb)
    with sw.Plan(pb) as plan:
        plan.eval(0, plan.n)
        _check_winners(plan.select_batch(pb.queries), g["winners"])
        assert plan.pareto() == [tuple(p) for p in g["front"]]
        assert plan.digest() == int(g["digest"])
        rng = random.Random(11)
        for _ in range(200):
            b = rng.randrange(plan.n - 512)
            _records_equal(plan, orc, b, b + 512)
        _records_equal(plan, orc, plan.n - 512, plan.n)


def test_ragged_subrange_and_split_invariance(sw, oracle_mod):
    pb = make_config("C2")
    orc = oracle_mod.Oracle(pb)
    b, e = 123_457, 123_457 + 1_500_001
    qs = pb.queries + [Query(200_000_000, 10**9, 3_000_000)]
    w, f, d = orc.sweep(b, e, qs)
    exp = [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]
    with sw.Plan(pb, record_capacity=e - b) as plan:
        plan.eval(b, e)
        _check_winners(plan.select_batch(qs), exp)
        assert plan.pareto() == f
        assert plan.digest() == d
    with sw.Plan(pb, record_capacity=e - b) as plan:  # same range in 3 ragged calls
        m1, m2 = b + 333_333, b + 1_000_003
        plan.eval(m1, m2)
        plan.eval(b, m1)
        plan.eval(m2, e)
        _check_winners(plan.select_batch(qs), exp)
        assert plan.pareto() == f
        assert plan.digest() == d


def test_shard_emulation_single_gpu(sw, oracle_mod):
    """Rank shards computed by sw_shard_range, each evaluated by its own handle, union
    equals the whole space (records partition it, digests add up)."""
    pb = make_config("C3")
    row = None
    total = 0
    digests = 0
    with sw.Plan(pb, record_capacity=1) as p0:
        row, n = p0.row, p0.n
    b0, e0 = 7, n - 5
    prev = b0
    for r in range(4):
        b, e = sw.shard_range(b0, e0, row, r, 4)
        assert b == prev
        prev = e
        with sw.Plan(pb, record_capacity=e - b) as plan:
            plan.eval(b, e)
            digests += plan.digest()
            total += e - b
    assert prev == e0 and total == e0 - b0
    # oracle digest over [7, n-5) = full digest minus the 12 excluded records
    g = _golden("C3")
    rest = orc_rest = oracle_mod.Oracle(pb)
    ex = sum(orc_rest.record_hash(i, r) for i, r in
             list(enumerate(rest.record_list(0, 7))) + [(n - 5 + j, r) for j, r in enumerate(rest.record_list(n - 5, n))])
    assert (digests + ex) % (1 << 64) == int(g["digest"])


def test_error_paths(sw):
    pb = make_config("C1")
    bad = make_config("C1")
    bad.choices = [(1, 3, 0)] + bad.choices[1:]  # k = 3 > G = 2
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(bad)
    assert ei.value.status == sw.SW_EINVAL
    bad = make_config("C1")
    bad.dur_us = [0] + bad.dur_us[1:]
    with pytest.raises(sw.SwError):
        sw.Plan(bad)
    with sw.Plan(pb, record_capacity=100) as plan:
        plan.eval(0, 100)
        with pytest.raises(sw.SwError) as ei:
            plan.eval(50, 60)  # overlap
        assert ei.value.status == sw.SW_EINVAL
        with pytest.raises(sw.SwError) as ei:
            plan.eval(100, 256)  # capacity
        assert ei.value.status == sw.SW_ERANGE
        with pytest.raises(sw.SwError):
            plan.eval(0, 257)
        plan.reset()
        plan.eval(100, 200)  # after reset the front persists, records are new
    with sw.Plan(pb) as plan:
        s = plan.select()
        assert s.status == sw.SW_EMPTY


def test_fleet_c4(sw):
    g = _golden("C4")
    fleet = make_fleet()
    for pb, gr in zip(fleet, g["requests"]):
        with sw.Plan(pb) as plan:
            plan.eval(0, plan.n)
            _check_winners(plan.select_batch(pb.queries), gr["winners"])
            assert plan.digest() == int(gr["digest"])
            assert plan.pareto() == [tuple(p) for p in gr["front"]]
