"""Multi-rank parity on ONE GPU: R in {2, 4, 8} emulated ranks.

Each rank is a handle driven by its own host thread, connected by the library's loopback
communicator (sw_comm_loopback_create): the collectives are enqueued on each handle's
stream with NCCL's ordering, so the multi-rank code path -- sharded eval, per-rank scans,
the allgather of winners + select_final_kernel merge, the padded front allgather +
front_gather_pad_kernel + cooperative Pareto merge, the digest allreduce, the status-word
reduction -- runs unchanged on a one-GPU box.  Every result is compared with the oracle
(tests/golden/, written by tools/gen_golden.py from oracle/ only); the merge must preserve
the objective, the closest tier and the exact front.
"""
import json
import os
import threading

import pytest

from swgen import make_config, make_fleet
from swgen.generator import Query
from tests.conftest import cuda_available

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


def run_ranks(sw, R, fn, timeout=600):
    """fn(rank, comm) on R threads over one loopback group -> per-rank results."""
    comms = sw.comm_loopback_create(R)
    res, errs = [None] * R, [None] * R

    def work(r):
        try:
            res[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errs[r] = e
    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
        assert not t.is_alive(), "loopback rank hung"
    for c in comms:
        sw.comm_destroy(c)
    return res, errs


def _check(sels, front, dg, g):
    for s, w in zip(sels, g["winners"]):
        st = {0: 0, 1: 1, -1: 3}[w["status"]]
        assert s.status == st, (s, w)
        assert s.index == w["index"] and tuple(s.rec) == tuple(w["rec"]), (s, w)
    assert front == [tuple(p) for p in g["front"]]
    assert dg == int(g["digest"])


@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_loopback_eval_select_front_digest(sw, cfg, R):
    """Global range in two ragged calls, every rank shards both internally; winners,
    front and digest on EVERY rank equal the oracle's full sweep."""
    pb = make_config(cfg)
    g = _golden(cfg)

    def rank(r, comm):
        with sw.Plan(pb, device=0, comm=comm, rank=r, nranks=R) as plan:
            cut = plan.n // 3 + 12345
            plan.eval(cut, plan.n)
            plan.eval(0, cut)
            sels = plan.select_batch(pb.queries)
            front = plan.pareto()
            dg = plan.digest()
            # per-rank shards partition the space
            segs = plan.segments()
        return sels, front, dg, segs
    res, errs = run_ranks(sw, R, rank)
    assert not any(errs), errs
    for sels, front, dg, _ in res:
        _check(sels, front, dg, g)
    # the rank shards of each call are disjoint and cover it
    for call in range(2):
        spans = sorted((x[3][call]["shard_begin"], x[3][call]["shard_end"]) for x in res)
        lo, hi = res[0][3][call]["global_begin"], res[0][3][call]["global_end"]
        assert spans[0][0] == lo and spans[-1][1] == hi
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.parametrize("R", [2, 4])
def test_loopback_sweep_and_stream(sw, R):
    """The chunked sweep (per-chunk winners merged, running front) and the fused stream
    mode (no records; per-rank candidate lists merged) at R ranks on C3."""
    pb = make_config("C3")
    g = _golden("C3")

    def rank(r, comm):
        with sw.Plan(pb, device=0, comm=comm, rank=r, nranks=R, record_capacity=30_000_000) as plan:
            sels, dg = plan.sweep(0, plan.n, pb.queries, digest=True)
            front = plan.pareto()
        with sw.Plan(pb, device=0, comm=comm, rank=r, nranks=R, record_capacity=1024) as plan:
            ss = plan.stream(0, plan.n, pb.queries)
            sf = plan.pareto()
        return sels, front, dg, ss, sf
    res, errs = run_ranks(sw, R, rank)
    assert not any(errs), errs
    for sels, front, dg, ss, sf in res:
        _check(sels, front, dg, g)
        _check(ss, sf, int(g["digest"]), g)


def test_loopback_fleet(sw):
    """sw_fleet_* over 2 ranks: one allgather of the n winners, replicated merge (C4's
    first 24 requests, every winner vs the oracle golden)."""
    g = _golden("C4")
    fleet = make_fleet()[:24]

    def rank(r, comm):
        with sw.Fleet(fleet, device=0, comm=comm, rank=r, nranks=2) as F:
            F.eval()
            return F.select([pb.queries[0] for pb in fleet])
    res, errs = run_ranks(sw, 2, rank)
    assert not any(errs), errs
    for sels in res:
        for s, gr in zip(sels, g["requests"][:24]):
            w = gr["winners"][0]
            assert s.status == {0: 0, 1: 1, -1: 3}[w["status"]]
            assert s.index == w["index"] and tuple(s.rec) == tuple(w["rec"])


def test_loopback_overflow_on_one_rank(sw, monkeypatch):
    """a survivor overflow on ONE rank must send every rank through the
    exact front redo together (the decision is taken on the status words reduced over the
    ranks).  SW_SURV_CAP=4096@0 shrinks rank 0's survivor buffer only; the front-answered
    query (R30) and the front still equal the oracle's on both ranks."""
    monkeypatch.setenv("SW_SURV_CAP", "4096@0")
    pb = make_config("C3")
    g = _golden("C3")

    def rank(r, comm):
        with sw.Plan(pb, device=0, comm=comm, rank=r, nranks=2) as plan:
            plan.eval(0, plan.n)
            sels = plan.select_batch(pb.queries)
            return sels, plan.pareto(), plan.digest()
    res, errs = run_ranks(sw, 2, rank)
    assert not any(errs), errs
    for sels, front, dg in res:
        _check(sels, front, dg, g)


def test_loopback_mismatched_calls(sw):
    """Ranks that make different select calls fail together with SW_ESTATE (no hang, no
    silently wrong answer on either rank)."""
    pb = make_config("C1")

    def rank(r, comm):
        with sw.Plan(pb, device=0, comm=comm, rank=r, nranks=2) as plan:
            plan.eval(0, plan.n)
            q = Query(30_000_000 + r, 0, 1 << 62)  # rank-dependent SLO: a different call
            try:
                plan.select_batch([q])
            except sw.SwError as e:
                return e.status
            return 0
    res, errs = run_ranks(sw, 2, rank)
    assert not any(errs), errs
    assert res == [sw.SW_ESTATE, sw.SW_ESTATE]
