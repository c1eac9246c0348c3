"""World-size-2 gloo checks of the multi-rank HOST logic, no GPU.

Each rank takes the shard ``sw_shard_range`` gives it (row size from
``sw_space_shape``), computes its shard's winners / front / digest with the CPU
oracle (test infrastructure standing in for the per-rank GPU results), the ranks
exchange them over torch.distributed (gloo), and the library's host merge
``sw_selection_merge`` combines the winners.  The merged result must equal the
oracle's sweep of the whole range: the sharding partitions the space, the merge is
the query's total order (R13), and it is associative and commutative.
"""
import os
import random
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from swgen import make_config, INF
from swgen.generator import Query
from tests.helpers import random_problem

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problems():
    out = [(make_config("C1"), 0, None)]
    c3 = make_config("C3")
    out.append((c3, 1_234_567, 1_234_567 + 300_011))  # ragged sub-range of C3
    for seed in range(6):
        rng = random.Random(77 + seed)
        pb = random_problem(rng, max_scenes=6, max_pools=3, max_choices=5,
                            one_scene_digits=rng.random() < 0.5)
        pb.queries = [Query(INF, INF, INF),
                      Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**6)),
                      Query(0, 0, 0)]
        out.append((pb, 0, None))
    return out


def _to_sel(sw, w, n_pools, B):
    st, idx, rec = w
    status = {0: sw.SW_OK, 1: sw.SW_CLOSEST, -1: sw.SW_EMPTY}[st]
    return sw.Selection(status, idx if st != -1 else 0, rec.astuple() if st != -1 else (0,) * 6,
                        0, 0, [0] * n_pools, [0] * B)


def _worker(rank, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        import paper_2603_05800_b200 as sw
        from oracle.oracle import Oracle, pareto_points
        for pb, b0, e0 in _problems():
            orc = Oracle(pb)
            n, row = sw.space_shape(pb)
            assert n == orc.n
            e0 = n if e0 is None else e0
            b, e = sw.shard_range(b0, e0, row, rank, WORLD)
            w, f, d = orc.sweep(b, e, pb.queries, nthreads=2)
            mine = {"range": (b, e), "winners": w, "front": f, "digest": d}
            got = [None] * WORLD
            dist.all_gather_object(got, mine)
            # the shards partition [b0, e0) in rank order, row-aligned inside
            assert got[0]["range"][0] == b0 and got[-1]["range"][1] == e0
            for r in range(WORLD - 1):
                assert got[r]["range"][1] == got[r + 1]["range"][0]
            for r in range(1, WORLD):
                lo = got[r]["range"][0]
                assert lo == e0 or lo % row == 0
            W, F, Dg = orc.sweep(b0, e0, pb.queries, nthreads=2)
            P, B = len(pb.gpus), len(pb.radix)
            for qi, q in enumerate(pb.queries):
                sels = [_to_sel(sw, g["winners"][qi], P, B) for g in got]
                fwd = sels[0]
                for s in sels[1:]:
                    fwd = sw.selection_merge(pb.objective, q, fwd, s)
                rev = sels[-1]
                for s in reversed(sels[:-1]):
                    rev = sw.selection_merge(pb.objective, q, s, rev)
                exp = _to_sel(sw, W[qi], P, B)
                for m in (fwd, rev):
                    assert m.status == exp.status, (pb.name, qi, m, exp)
                    if exp.status != sw.SW_EMPTY:
                        assert m.index == exp.index and tuple(m.rec) == tuple(exp.rec)
            # digest is additive mod 2^64; the front of the union of the rank fronts
            # equals the front of the whole range (front(A u B) = front(fA u fB))
            assert sum(g["digest"] for g in got) % (1 << 64) == Dg
            union = [p for g in got for p in g["front"]]
            assert sorted(pareto_points(union), key=lambda p: (p[1], p[2], -p[3], p[0])) == F
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as ex:  # report to the parent
        import traceback
        errq.put("rank %d: %s\n%s" % (rank, ex, traceback.format_exc()))
        raise


def test_two_rank_shard_and_merge_gloo():
    from paper_2603_05800_b200 import build
    build.build()
    from oracle import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, errq)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_selection_merge_rules():
    """Hand cases of the total order: feasible beats closest, lower index breaks ties,
    EMPTY loses, COST_X_TTFF compares the 128-bit product."""
    import paper_2603_05800_b200 as sw
    S = sw.Selection
    q = Query(100, 0, 1000)
    feas = S(sw.SW_OK, 9, (50, 0, 900, 10, 0, 1), 0, 0, [0], [0])
    feas_hi_q = S(sw.SW_OK, 12, (60, 0, 950, 20, 0, 1), 0, 0, [0], [0])
    close = S(sw.SW_CLOSEST, 1, (150, 0, 10, 99, 0, 1), 0, 0, [0], [0])
    empty = S(sw.SW_EMPTY, 0, (0,) * 6, 0, 0, [0], [0])
    assert sw.selection_merge(0, q, close, feas).index == 9
    assert sw.selection_merge(0, q, feas, feas_hi_q).index == 12   # higher quality first
    assert sw.selection_merge(0, q, empty, close).status == sw.SW_CLOSEST
    assert sw.selection_merge(0, q, empty, empty).status == sw.SW_EMPTY
    twin = S(sw.SW_OK, 3, feas.rec, 0, 0, [0], [0])
    assert sw.selection_merge(0, q, feas, twin).index == 3          # equal keys: lower index
    # closest tier: smaller startup+stall violation wins, then smaller budget violation
    c1 = S(sw.SW_CLOSEST, 5, (120, 0, 5000, 10, 0, 1), 0, 0, [0], [0])
    c2 = S(sw.SW_CLOSEST, 6, (110, 0, 9000, 10, 0, 1), 0, 0, [0], [0])
    assert sw.selection_merge(0, q, c1, c2).index == 6
    # COST_X_TTFF: 2^40 * 2^30 overflows 64 bits; compare as 128-bit
    big = S(sw.SW_OK, 1, (1 << 30, 0, 1 << 40, 0, 0, 1), 0, 0, [0], [0])
    small = S(sw.SW_OK, 2, ((1 << 30) - 1, 0, 1 << 40, 0, 0, 1), 0, 0, [0], [0])
    qi = Query(INF, INF, INF)
    assert sw.selection_merge(1, qi, big, small).index == 2
    with pytest.raises(sw.SwError):
        sw.selection_merge(2, qi, big, small)
