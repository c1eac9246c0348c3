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
    for cfg in ["C1", "C2", "C3", "C3w", "C3s", "C3t", "C3u", "C5"]:
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


@pytest.mark.parametrize("cfg", ["C2", "C3", "C2x"])
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


def test_c5_chunked_sweep(sw):
    """C5 (48^6 = 1.2e10 plans, 60 scenes, 3 pools) on the oracle's pinned sub-ranges,
    through sw_plan_sweep with a record buffer far smaller than the range (7 chunks):
    winners (merged across chunks), digest and the running front."""
    g = _golden("C5sub")
    pb = make_config("C5")
    for rg in g["ranges"]:
        b, e = rg["begin"], rg["end"]
        with sw.Plan(pb, record_capacity=8_000_000) as plan:
            sels, dg = plan.sweep(b, e, pb.queries, digest=True)
            _check_winners(sels, rg["winners"])
            assert dg == int(rg["digest"])
            assert plan.pareto() == [tuple(p) for p in rg["front"]]
            # winners carry their full detail (recomputed on the GPU)
            for s in sels:
                d, _ = plan.detail(s.index)
                assert tuple(d.rec) == tuple(s.rec) and d.digit == s.digit


def test_sweep_matches_eval_select(sw, oracle_mod):
    """sw_plan_sweep over ragged chunks == one eval + select_batch + pareto (C3 sub-range)."""
    pb = make_config("C3")
    b, e = 5_000_003, 5_000_003 + 2_345_679
    orc = oracle_mod.Oracle(pb)
    w, f, d = orc.sweep(b, e, pb.queries)
    exp = [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]
    with sw.Plan(pb, record_capacity=600_000) as plan:
        sels, dg = plan.sweep(b, e, pb.queries, chunk=511_111, digest=True)
        _check_winners(sels, exp)
        assert dg == d
        assert plan.pareto() == f
        with pytest.raises(sw.SwError):  # chunk larger than the capacity allows
            plan.sweep(0, 10, pb.queries, chunk=10**9)
        plan.eval(0, 1000)
        with pytest.raises(sw.SwError) as ei:  # records held: sweep refuses
            plan.sweep(2000, 3000, pb.queries)
        assert ei.value.status == sw.SW_ESTATE


def test_interleaved_handles(sw, oracle_mod):
    """Handles with different table sizes created first, evaluated after (per-kernel
    launch attributes must not leak between handles); each matches the oracle."""
    probs = [make_config("C1"), make_config("C3"), make_config("C1")]
    probs[1].name = "C3"
    plans = [sw.Plan(pb, record_capacity=200_000) for pb in probs]
    try:
        for p in plans:
            p.eval(0, min(p.n, 200_000))
        for pb, p in zip(probs, plans):
            n = min(p.n, 200_000)
            orc = oracle_mod.Oracle(pb)
            w, f, d = orc.sweep(0, n, pb.queries)
            _check_winners(p.select_batch(pb.queries),
                           [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w])
            assert p.digest() == d
    finally:
        for p in plans:
            p.close()


def test_fleet_batch_api(sw):
    """C4 through sw_fleet_*: one eval launch for all 256 requests, one select scan with
    per-request SLO/budget; every winner, every digest and a sample of fronts vs the
    oracle golden; reset + second round gives the same winners."""
    g = _golden("C4")
    fleet = make_fleet()
    with sw.Fleet(fleet) as F:
        for rnd in range(2):
            if rnd:
                F.reset()
            F.eval()
            sels = F.select([pb.queries[0] for pb in fleet])
            for s, gr in zip(sels, g["requests"]):
                _check_winners([s], gr["winners"])
        for i, (pb, gr) in enumerate(zip(fleet, g["requests"])):
            p = F.plan(i)
            assert p.digest() == int(gr["digest"]), i
            if i % 16 == 5:
                assert p.pareto() == [tuple(x) for x in gr["front"]], i
            d, _ = p.detail(sels[i].index)
            assert tuple(d.rec) == tuple(sels[i].rec) and d.digit == sels[i].digit
        assert F.launch_count() > 0


def test_decode_and_segments(sw, oracle_mod):
    """sw_plan_decode (host helper) == the oracle's decoder, per scene; sw_plan_segments
    describes the tiled layout: every record read through the zero-copy view's slot
    formula equals the oracle's record."""
    import ctypes
    pb = make_config("C3")
    orc = oracle_mod.Oracle(pb)
    rng = random.Random(3)
    with sw.Plan(pb, record_capacity=3_000_000) as plan:
        for _ in range(50):
            i = rng.randrange(plan.n)
            dig = orc.decode(i)
            per_scene = plan.decode(i)
            for b in range(len(pb.radix)):
                for s_ in range(pb.first_scene[b], pb.first_scene[b + 1]):
                    assert per_scene[s_] == dig[b]
        plan.eval(1_000_003, 2_000_005)
        plan.eval(17, 400_000)
        segs = plan.segments()
        assert [(x["global_begin"], x["global_end"]) for x in segs] == [(1_000_003, 2_000_005), (17, 400_000)]
        ptr, nslots = plan.records_view()
        from paper_2603_05800_b200._native import sw_record
        rt = _cudart()
        for sg in segs:
            for i in [sg["shard_begin"], sg["shard_end"] - 1] + [rng.randrange(sg["shard_begin"], sg["shard_end"])
                                                                   for _ in range(30)]:
                H, j = divmod(i, sg["row"])
                slot = sg["offset"] + ((H // 32 - sg["tile0"]) * sg["row"] + j) * 32 + H % 32
                assert slot < nslots
                buf = (ctypes.c_uint8 * 32)()
                assert rt.cudaMemcpy(ctypes.c_void_p(ctypes.addressof(buf)), ctypes.c_void_p(ptr + 32 * slot),
                                     ctypes.c_size_t(32), 2) == 0  # cudaMemcpyDeviceToHost
                rec = sw_record.from_buffer_copy(buf)
                assert rec.astuple() == orc.records(i, i + 1)[0].astuple(), i


def _cudart():
    """The CUDA runtime (torch's copy) through ctypes, to read the zero-copy view."""
    import ctypes
    import glob
    import torch
    torch.cuda.init()
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            pass
    import nvidia.cuda_runtime
    d = os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib")
    return ctypes.CDLL(sorted(glob.glob(os.path.join(d, "libcudart.so*")))[0])


@pytest.mark.parametrize("cfg", ["C3d", "C3e", "C3ex"])
def test_disagg_and_energy_full_space(sw, oracle_mod, cfg):
    """C3d (FramePack DiT/VAE disaggregated onto a VAE pool, R37) and
    C3e / C3ex (records scored by energy in microjoules, QUALITY_FIRST and Energy x TTFF,
    R38): the full space at the bench's launch configuration -- winners, exact front,
    digest -- plus sampled records and winner details vs the oracle."""
    pb = make_config(cfg)
    g = _golden(cfg)
    orc = oracle_mod.Oracle(pb)
    with sw.Plan(pb) as plan:
        plan.eval(0, plan.n)
        sels = plan.select_batch(pb.queries)
        _check_winners(sels, g["winners"])
        assert plan.pareto() == [tuple(p) for p in g["front"]]
        assert plan.digest() == int(g["digest"])
        rng = random.Random(13)
        for _ in range(40):
            b = rng.randrange(plan.n - 512)
            _records_equal(plan, orc, b, b + 512)
        for _ in range(10):
            i = rng.randrange(plan.n)
            sel, ready = plan.detail(i)
            rec, oready, pend, mk, te = orc.eval(i)
            assert tuple(sel.rec) == rec.astuple() and ready == oready and sel.pool_end_us == pend


@pytest.mark.parametrize("seed", range(6))
def test_disagg_energy_random(sw, oracle_mod, seed):
    """Random problems with VAE stages on a VAE pool and/or the energy metric (both
    billings, both objectives): every record, winners, front, digest; stream == records."""
    from tests.test_disagg_energy_oracle import _disagg
    rng = random.Random(2000 + seed)
    pb = random_problem(rng, max_scenes=6, max_pools=3, max_choices=4, one_scene_digits=rng.random() < 0.5)
    if seed % 3 != 2:
        _disagg(pb, rng)
    if seed % 3 != 0:
        pb.metric = 1
        pb.power_active_w = [rng.randint(200, 1200) for _ in pb.gpus]
        pb.power_idle_w = [rng.randint(10, 150) for _ in pb.gpus]
    orc = oracle_mod.Oracle(pb)
    n = orc.n
    qs = [Query(INF, INF, INF), Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**12)),
          Query(0, 0, 0)]
    w, f, d = orc.sweep(0, n, qs)
    exp = [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]
    with sw.Plan(pb) as plan:
        plan.eval(0, n)
        _records_equal(plan, orc, 0, n)
        _check_winners(plan.select_batch(qs), exp)
        assert plan.pareto() == f
        assert plan.digest() == d
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(0, n, qs), exp)
        assert plan.pareto() == f


def test_c5_full_space(sw):
    """C5 (48^6 = 1.2e10 plans, 391 GB of records) over the WHOLE space through the chunked
    sweep at the bench's launch configuration (records capacity 75% of free HBM): winners,
    exact front and digest vs the oracle's full-space result (computed once in pieces and
    cached by input SHA-256, tools/gen_golden_full.py)."""
    g = _golden("C5")
    import torch
    pb = make_config("C5")
    sw.trim_device_memory(0)
    free_b, _ = torch.cuda.mem_get_info(0)
    cap = int(0.75 * free_b) // 32
    with sw.Plan(pb, record_capacity=cap) as plan:
        sels, dg = plan.sweep(0, plan.n, pb.queries, digest=True)
        _check_winners(sels, g["winners"])
        assert dg == int(g["digest"])
        assert plan.pareto() == [tuple(p) for p in g["front"]]
