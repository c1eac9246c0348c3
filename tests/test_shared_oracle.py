"""Pins of the shared-pool fleet oracle (reading R36).

or_shared_eval simulates every shared pool as an online, non-preemptive EDF queue of gang
tasks ("model instances maintain local queues that prioritize tasks by
deadline").  It is pinned, independently of its own code, by:
  - reduction to the single-request recurrence (itself pinned in test_oracle_pins.py);
  - disjoint pools = independent requests;
  - a hand-worked two-request example (the early scene of a NEW request overtakes the
    later scene of an earlier request) and its batch variant;
  - a time-stepped brute-force simulation (a different algorithm) on tiny inputs;
  - the 1/3 real-time, 1/3 relaxed, 1/3 batch mix on SF3.
"""
import random

import pytest

from swgen import make_shared, SharedFleet, INF
from swgen.generator import Query
from tests.helpers import make_problem, random_problem

M64 = (1 << 64) - 1


def _sf(reqs, arrivals, slo_t, slo_s, fixed=None, gpus=None, price=None, billing=0):
    gpus = gpus or reqs[0].gpus
    price = price or reqs[0].price_mc
    for pb in reqs:
        pb.gpus, pb.price_mc, pb.billing = list(gpus), list(price), billing
    return SharedFleet("t", reqs, list(arrivals), list(slo_t), list(slo_s),
                       fixed or [None] * len(reqs), list(gpus), list(price), billing=billing)


def _sat(x, y):
    return x - y if x > y else 0


def test_single_request_reduces_to_recurrence(oracle_mod):
    """One request alone on the pools: the EDF fleet simulation gives the single-request
    recurrence's ready times and metrics (shifted by the arrival), every candidate."""
    rng = random.Random(401)
    n = 0
    for trial in range(60):
        pb = random_problem(rng, max_scenes=5, max_pools=3, max_choices=3,
                            one_scene_digits=rng.random() < 0.5)
        pb.billing = rng.randrange(2)
        T0 = rng.choice([0, 0, rng.randint(1, 10**7)])
        st, ss = rng.choice([INF, rng.randint(0, 10**8)]), rng.choice([INF, rng.randint(0, 10**8)])
        sf = _sf([pb], [T0], [st], [ss], billing=pb.billing)
        so = oracle_mod.SharedOracle(sf)
        o = oracle_mod.Oracle(pb)
        assert so.n == o.n
        for i in range(o.n):
            rec, ready, pend, mk, te = o.eval(i)
            f, per, rd = so.eval(i)
            r = per[0]
            assert (r.ttff_us, r.stall_us, r.quality, r.stall_count) == \
                (rec.ttff_us, rec.stall_us, rec.quality, rec.stall_count)
            assert [x - T0 for x in rd[0]] == ready
            assert (f.ttff_us, f.stall_us) == (_sat(rec.ttff_us, st), _sat(rec.stall_us, ss))
            assert (f.quality, f.stall_count, f.flags) == (rec.quality, rec.stall_count, rec.flags)
            if T0 == 0:
                assert f.cost_mc == rec.cost_mc
            n += 1
    assert n > 500


def test_disjoint_pools_are_independent(oracle_mod):
    """Requests that never share a pool do not interact: each request's metrics equal its
    solo evaluation; at equal arrival 0 the fleet cost is the sum of the solo costs."""
    rng = random.Random(402)
    for trial in range(30):
        reqs = []
        for r in range(2):
            pb = random_problem(rng, max_scenes=4, max_pools=1, max_choices=3)
            reqs.append(pb)
        g = [reqs[0].gpus[0], reqs[1].gpus[0]]
        price = [reqs[0].price_mc[0], reqs[1].price_mc[0]]
        reqs[1].choices = [(l, k, 1) for (l, k, p) in reqs[1].choices]  # request 1 on pool 1
        solo = []
        for r, pb in enumerate(reqs):
            pb2 = make_problem(pb.dur_us, pb.llm_us, pb.tts_us, g, price, pb.radix, pb.first_scene,
                               pb.choices, pb.va_us, overhead_us=pb.overhead_us,
                               fixed_cost_mc=pb.fixed_cost_mc, billing=0, heads=0)
            solo.append(oracle_mod.Oracle(pb2))
        sf = _sf(reqs, [0, 0], [INF, INF], [INF, INF], gpus=g, price=price)
        so = oracle_mod.SharedOracle(sf)
        n1 = solo[1].n
        for i in rng.sample(range(so.n), min(so.n, 40)):
            f, per, rd = so.eval(i)
            i0, i1 = divmod(i, n1)
            r0 = solo[0].eval(i0)[0]
            r1 = solo[1].eval(i1)[0]
            for r, x in zip(per, (r0, r1)):
                assert (r.ttff_us, r.stall_us, r.quality, r.stall_count) == \
                    (x.ttff_us, x.stall_us, x.quality, x.stall_count)
            assert f.cost_mc == r0.cost_mc + r1.cost_mc


def _hand_fleet(slo_b):
    # one pool of 1 GPU, price 3.6e9 mc per GPU-hour = 1 mc per GPU-us (exact)
    A = make_problem([1_000_000, 1_000_000], [10, 10], [0, 0], [1], [3_600_000_000], [1, 1], [0, 1, 2],
                     [(0, 1, 0), (0, 1, 0)], [100, 100], heads=0)
    B = make_problem([1_000_000], [10], [0], [1], [3_600_000_000], [1], [0, 1], [(0, 1, 0)], [5], heads=0)
    return _sf([A, B], [0, 30], [50, slo_b], [0, 0])


def test_hand_worked_two_request_edf(oracle_mod):
    """"the image generation model may process an early scene from a new request
    before a later scene from an earlier request if it has a tighter deadline".
    A (arrives 0): scenes released at 10 and 20 us (LLM 10 us each), 100 us of video each,
    SLO 50 us -> deadlines 50 and 1,000,050.  B (arrives 30): its scene released at 40,
    5 us, SLO 5 -> deadline 35.  One GPU.  By hand: A0 starts at 10 (only task), ends 110;
    at 20 A1 is head but the GPU is busy until 110, and B0 (deadline 35 < 1,000,050) is
    released at 40 <= 110, so B0 takes the decision: 110-115; then A1: 115-215.
    A: ttff 110, stall 0; B: ttff 115 - 30 = 85.  Fleet: startup lateness
    max(110 - 50, 85 - 5) = 80, stall lateness 0, cost = 215 GPU-us at 1 mc/GPU-us
    = floor(215.5) = 215 mc, Q = 3 scenes x 1000 ms x 250."""
    so = oracle_mod.SharedOracle(_hand_fleet(5))
    f, per, rd = so.eval(0)
    assert rd == [[110, 215], [115]]
    assert (per[0].ttff_us, per[0].stall_us, per[1].ttff_us, per[1].stall_us) == (110, 0, 85, 0)
    assert (f.ttff_us, f.stall_us, f.cost_mc, f.quality, f.stall_count, f.flags) == (80, 0, 215, 750_000, 0, 1)


def test_hand_worked_batch_yields_nothing(oracle_mod):
    """Same fleet with B a batch request (no SLO): its deadline is infinite,
    A1 keeps the GPU (110-210) and B0 runs last (210-215): B ttff 185, no lateness."""
    so = oracle_mod.SharedOracle(_hand_fleet(INF))
    f, per, rd = so.eval(0)
    assert rd == [[110, 210], [215]]
    assert per[1].ttff_us == 185
    assert (f.ttff_us, f.stall_us, f.cost_mc) == (60, 0, 215)


def _time_stepped(sf, plans):
    """Brute force by a different algorithm: advance time one microsecond at a time; at
    each instant every pool starts its EDF head (smallest (deadline, request, scene) among
    released unstarted tasks) if k of its GPUs are free, and repeats; any free GPUs serve
    (decisions never go back in time, so which free GPU is taken is immaterial)."""
    tasks = []
    ready = {}
    for r, (pb, pl) in enumerate(zip(sf.requests, plans)):
        a, L, A = [], pb.overhead_us, 0
        for s in range(pb.S):
            L += pb.llm_us[s]
            A = max(L, A) + pb.tts_us[s]
            a.append(A)
        P = [sum(pb.dur_us[:s]) for s in range(pb.S)]
        digs, x = [], pl
        for rad in reversed(pb.radix):
            digs.append(x % rad)
            x //= rad
        digs.reverse()
        coff = [sum(pb.radix[:b]) for b in range(pb.B)]
        for s in range(pb.S):
            b = max(bb for bb in range(pb.B) if pb.first_scene[bb] <= s)
            lv, k, p = pb.choices[coff[b] + digs[b]]
            t = pb.va_us[pb.va_offset(b) + (s - pb.first_scene[b]) * pb.radix[b] + digs[b]]
            dl = M64 if sf.slo_startup_us[r] == INF else sf.arrival_us[r] + sf.slo_startup_us[r] + P[s]
            tasks.append(dict(r=r, s=s, k=k, p=p, t=t, rel=sf.arrival_us[r] + a[s], dl=dl))
    for p, G in enumerate(sf.gpus):
        busy_until = [0] * G
        todo = [x for x in tasks if x["p"] == p]
        tm = 0
        while todo:
            while True:
                rel = [x for x in todo if x["rel"] <= tm]
                if not rel:
                    break
                h = min(rel, key=lambda x: (x["dl"], x["r"], x["s"]))
                free = [g for g in range(G) if busy_until[g] <= tm]
                if len(free) < h["k"]:
                    break
                for g in free[: h["k"]]:
                    busy_until[g] = tm + h["t"]
                ready[(h["r"], h["s"])] = tm + h["t"]
                todo.remove(h)
            tm += 1
    return ready


def test_matches_time_stepped_brute_force(oracle_mod):
    rng = random.Random(403)
    for trial in range(40):
        reqs = []
        P = rng.randint(1, 2)
        gpus = [rng.randint(1, 3) for _ in range(P)]
        for r in range(rng.randint(2, 3)):
            S = rng.randint(1, 3)
            dur = [rng.randint(1, 30) * 1000 for _ in range(S)]
            ch = []
            for _ in range(2):
                p = rng.randrange(P)
                ch.append((rng.randrange(4), rng.randint(1, gpus[p]), p))
            va = [rng.randint(1, 40) for _ in range(2 * S)]
            pb = make_problem(dur, [rng.randint(0, 15) for _ in range(S)], [rng.randint(0, 5) for _ in range(S)],
                              gpus, [180250] * P, [2] * S, list(range(S + 1)), ch * S, va, heads=0)
            reqs.append(pb)
        R = len(reqs)
        sf = _sf(reqs, [rng.randint(0, 40) for _ in range(R)],
                 [rng.choice([INF, rng.randint(0, 60)]) for _ in range(R)], [INF] * R)
        so = oracle_mod.SharedOracle(sf)
        for i in rng.sample(range(so.n), min(so.n, 12)):
            plans = so.decode(i)
            exp = _time_stepped(sf, plans)
            _, _, rd = so.eval(i)
            for (r, s), e in exp.items():
                assert rd[r][s] == e, (trial, i, r, s)


def test_sf3_mix_real_time_first(oracle_mod):
    """SF3, the 1/3 real-time / 1/3 relaxed / 1/3 batch mix: the batch
    request's tasks live on the A100 pool, the real-time one's on the H100 pool; whenever
    the new (relaxed) request's plan keeps off the H100 pool, the real-time request runs
    exactly as it would alone -- sharing only couples requests through common pools."""
    sf = make_shared("SF3")
    so = oracle_mod.SharedOracle(sf)
    rng = random.Random(404)
    rt_alone = oracle_mod.SharedOracle(SharedFleet("rt", [sf.requests[0]], [0], [sf.slo_startup_us[0]],
                                                   [sf.slo_stall_us[0]], [sf.fixed_index[0]], sf.gpus, sf.price_mc))
    _, per_alone, rd_alone = rt_alone.eval(0)
    same = 0
    for i in rng.sample(range(so.n), 200):
        f, per, rd = so.eval(i)
        # the new request's plan never uses the H100 pool before the real-time one finishes
        # a scene released earlier -> when the new request keeps off pool 1 entirely, the
        # real-time request runs exactly as alone
        plan = so.decode(i)[2]
        pb = sf.requests[2]
        digs = []
        x = plan
        for rad in reversed(pb.radix):
            digs.append(x % rad)
            x //= rad
        pools = {pb.choices[sum(pb.radix[:b]) + d][2] for b, d in enumerate(reversed(digs))}
        if pools == {0}:
            assert rd[0] == rd_alone[0]
            same += 1
    assert same > 0
