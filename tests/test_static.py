"""STATIC rung for any scene ("If not enough, we switch to static content", P:823-825
"static elements (e.g., slides, ads) absorb latency"; reading R33): a
choice with degree k = 0 runs no video stage on no GPU, so the scene is ready once its text
and audio are, R_s = a_s, and contributes quality 0.

CPU part: the oracle pinned to closed forms (an all-STATIC plan: R_s = a_s, cost = the fixed
cost, Q = 0, no pool used, makespan = a_{S-1}) and to an equivalence that does not use the
STATIC code: a STATIC scene leaves every pool exactly as a private spare pool would, so the
other scenes' ready times equal those of the plan that sends the scene to a fresh extra
pool, whose own ready time is a_s + t.  GPU part: parity of the CUDA path with the oracle
on random problems with STATIC choices mixed in and on a ragged C3t sub-range.  Expected
values come only from oracle/ (live) or from those closed forms."""
import copy
import random

import pytest

from swgen import make_config, INF
from swgen.generator import Query
from tests.helpers import random_problem
from tests.test_gpu_parity import sw  # noqa: F401 (GPU fixture: skips without CUDA)


def _add_static(pb, rng, p_static=0.35):
    """Mix STATIC choices (level with score 0, k = 0, va_us = 0) into a problem's digits."""
    static_level = len(pb.level_score)
    pb.level_score = list(pb.level_score) + [0]
    choices, va, off, coff = [], [], 0, 0
    radix = []
    for b, r in enumerate(pb.radix):
        L = pb.first_scene[b + 1] - pb.first_scene[b]
        chs = list(pb.choices[coff:coff + r])
        rows = [pb.va_us[off + j * r: off + (j + 1) * r] for j in range(L)]
        if rng.random() < p_static:
            at = rng.randint(0, r)
            chs.insert(at, (static_level, 0, rng.randrange(len(pb.gpus))))
            for row in rows:
                row.insert(at, 0)
        choices.extend(chs)
        for row in rows:
            va.extend(row)
        radix.append(len(chs))
        off += L * r
        coff += r
    pb.radix, pb.choices, pb.va_us = radix, choices, va
    return pb


def _static_digit_values(pb):
    out, coff = [], 0
    for r in pb.radix:
        out.append([c for c in range(r) if pb.choices[coff + c][1] == 0])
        coff += r
    return out


def _index(radix, digits):
    i = 0
    for r, d in zip(radix, digits):
        i = i * r + d
    return i


def test_all_static_plan_closed_form(oracle_mod):
    """Every scene STATIC: R_s = a_s, cost = fixed cost, Q = 0, flags 0, makespan a_{S-1}."""
    rng = random.Random(3400)
    for _ in range(100):
        pb = _add_static(random_problem(rng, max_scenes=6, max_pools=3), rng, p_static=1.0)
        o = oracle_mod.Oracle(pb)
        a = o.fixed_stages()
        st = _static_digit_values(pb)
        i = _index(pb.radix, [c[0] for c in st])
        rec, ready, pend, mk, te = o.eval(i)
        s0 = pb.scene0_static
        assert ready[s0:] == a[s0:]
        assert rec.cost_mc == pb.fixed_cost_mc and rec.quality == 0 and rec.flags == 0
        assert list(pend) == [0] * len(pb.gpus)
        assert mk == max([ready[0]] + a[s0:])
        assert rec.ttff_us == ready[0]
        assert te == max(ready[s] - sum(pb.dur_us[:s]) for s in range(pb.S))


def test_static_scene_equals_private_spare_pool(oracle_mod):
    """A STATIC scene touches no pool: the plan's other ready times equal those of the plan
    that runs the scene on a fresh extra pool (k = 1 of S GPUs, t = 7 s), where it is ready
    at a_s + 7 s; its quality contribution is 0."""
    rng = random.Random(3401)
    for _ in range(150):
        pb = _add_static(random_problem(rng, max_scenes=6, max_pools=3), rng)
        st = _static_digit_values(pb)
        if not any(st):
            continue
        o = oracle_mod.Oracle(pb)
        a = o.fixed_stages()
        dig = [rng.randrange(r) for r in pb.radix]
        for b in range(len(dig)):
            if st[b] and rng.random() < 0.7:
                dig[b] = rng.choice(st[b])
        rec, ready, pend, mk, te = o.eval(_index(pb.radix, dig))
        # the same plan with every STATIC choice moved to a private pool of S GPUs (one
        # free GPU per scene, k = 1), t = 7 s
        alt = copy.deepcopy(pb)
        alt.gpus = list(pb.gpus) + [pb.S]
        alt.price_mc = list(pb.price_mc) + [0]
        alt.pool_class = list(pb.pool_class) + ["X"]
        extra = len(pb.gpus)
        alt.choices = [(l, 1, extra) if k == 0 else (l, k, p) for (l, k, p) in pb.choices]
        alt.va_us = [7_000_000 if v == 0 else v for v in pb.va_us]
        rec2, ready2, pend2, mk2, te2 = oracle_mod.Oracle(alt).eval(_index(alt.radix, dig))
        static_scenes = set()
        for b, d in enumerate(dig):
            if d in st[b]:
                static_scenes.update(range(pb.first_scene[b], pb.first_scene[b + 1]))
        for s in range(pb.S):
            if s in static_scenes:
                assert ready[s] == a[s] and ready2[s] == a[s] + 7_000_000
            else:
                assert ready[s] == ready2[s]
        assert list(pend) == list(pend2[:extra])
        assert rec.quality == rec2.quality  # STATIC scores 0 at both
        assert rec.flags == rec2.flags & ((1 << extra) - 1)


def test_c3t_config(oracle_mod):
    """C3t = C3 + a STATIC choice first in every digit: every plan of C3 keeps its record
    at digit values + 1."""
    a, b = make_config("C3"), make_config("C3t")
    assert b.radix == [r + 1 for r in a.radix]
    oa, ob = oracle_mod.Oracle(a), oracle_mod.Oracle(b)
    rng = random.Random(5)
    for _ in range(50):
        d = [rng.randrange(r) for r in a.radix]
        ra = oa.eval(_index(a.radix, d))[0]
        rb = ob.eval(_index(b.radix, [x + 1 for x in d]))[0]
        assert ra.astuple() == rb.astuple()


# ---------------------------------------------------------------- GPU parity


def _exp(w):
    return [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(10))
def test_gpu_random_problems_with_static(sw, oracle_mod, seed):  # noqa: F811
    from tests.test_gpu_parity import _check_winners, _records_equal
    rng = random.Random(3500 + seed)
    pb = random_problem(rng, max_scenes=7, max_pools=4, max_choices=5,
                        one_scene_digits=rng.random() < 0.5)
    pb = _add_static(pb, rng, p_static=0.6)
    if rng.random() < 0.4:
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


@pytest.mark.gpu
def test_gpu_c3t_subrange(sw, oracle_mod):  # noqa: F811
    """C3t: a ragged 3M sub-range (incl. the all-STATIC corner at index 0) through eval +
    select + front + digest and through the stream path; sampled records."""
    from tests.test_gpu_parity import _check_winners, _records_equal
    pb = make_config("C3t")
    orc = oracle_mod.Oracle(pb)
    for b, e in [(0, 1_500_007), (120_000_013, 123_000_029)]:
        w, f, d = orc.sweep(b, e, pb.queries)
        with sw.Plan(pb, record_capacity=e - b + 10**6) as plan:
            plan.eval(b, e)
            _check_winners(plan.select_batch(pb.queries), _exp(w))
            assert plan.pareto() == f
            assert plan.digest() == d
            rng = random.Random(13)
            for _ in range(20):
                x = rng.randrange(b, e - 256)
                _records_equal(plan, orc, x, x + 256)
        with sw.Plan(pb, record_capacity=1024) as plan:
            _check_winners(plan.stream(b, e, pb.queries), _exp(w))
            assert plan.pareto() == f
