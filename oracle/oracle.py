"""ctypes wrapper around oracle/sw_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this module.  The product package
(paper_2603_05800_b200) never does; it shares no code with this directory.
Inputs come from swgen (the seeded generator), which holds no method arithmetic.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sw_oracle.c")
LIB = os.path.join(HERE, "libsw_oracle.so")

U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)


class OrProblem(C.Structure):
    _fields_ = [
        ("S", C.c_uint32), ("dur_us", U64P), ("llm_us", U64P), ("tts_us", U64P),
        ("overhead_us", C.c_uint64), ("scene0_static", C.c_uint32),
        ("static_ready_us", C.c_uint64), ("n_pools", C.c_uint32), ("gpus", U32P),
        ("price_mc", U64P), ("fixed_cost_mc", C.c_uint64), ("billing", C.c_uint32),
        ("objective", C.c_uint32), ("n_levels", C.c_uint32), ("level_score", U32P),
        ("B", C.c_uint32), ("radix", U32P), ("first_scene", U32P),
        ("choice_level", U32P), ("choice_k", U32P), ("choice_pool", U32P),
        ("va_us", U64P), ("pool_ready_us", U64P), ("evict_risk_permille", U32P),
        ("vae_us", U64P), ("choice_vae_pool", U32P), ("metric", C.c_uint32),
        ("power_active_w", U32P), ("power_idle_w", U32P),
    ]


class OrRecord(C.Structure):
    _fields_ = [("ttff_us", C.c_uint64), ("stall_us", C.c_uint64), ("cost_mc", C.c_uint64),
                ("quality", C.c_uint32), ("stall_count", C.c_uint16), ("flags", C.c_uint8),
                ("pad", C.c_uint8)]

    def astuple(self):
        return (self.ttff_us, self.stall_us, self.cost_mc, self.quality, self.stall_count,
                self.flags)


class OrQuery(C.Structure):
    _fields_ = [("slo_startup_us", C.c_uint64), ("slo_stall_us", C.c_uint64),
                ("budget_mc", C.c_uint64)]


class OrWinner(C.Structure):
    _fields_ = [("index", C.c_uint64), ("rec", OrRecord), ("status", C.c_int32),
                ("pad", C.c_int32)]


class OrPoint(C.Structure):
    _fields_ = [("index", C.c_uint64), ("ttff_eff_us", C.c_uint64), ("cost_mc", C.c_uint64),
                ("quality", C.c_uint32), ("pad", C.c_uint32)]


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (building the checker is not using it)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-pthread", "-o", LIB, SRC])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.or_space_size.restype = C.c_uint64
        _lib.or_record_hash.restype = C.c_uint64
        _lib.or_pareto_points.restype = C.c_uint64
        _lib.or_sizeof_record.restype = C.c_uint32
        assert _lib.or_sizeof_record() == C.sizeof(OrRecord) == 32
        assert _lib.or_sizeof_point() == C.sizeof(OrPoint)
        assert _lib.or_sizeof_winner() == C.sizeof(OrWinner)
    return _lib


def _arr(ctype, vals):
    vals = list(vals)
    return (ctype * max(1, len(vals)))(*vals)


@dataclass
class Rec:
    ttff_us: int
    stall_us: int
    cost_mc: int
    quality: int
    stall_count: int
    flags: int

    @property
    def ttff_eff_us(self) -> int:
        return self.ttff_us + self.stall_us

    def astuple(self):
        return (self.ttff_us, self.stall_us, self.cost_mc, self.quality,
                self.stall_count, self.flags)


def _rec(r: OrRecord) -> Rec:
    return Rec(r.ttff_us, r.stall_us, r.cost_mc, r.quality, r.stall_count, r.flags)


class Oracle:
    """Holds the ctypes image of one swgen.Problem."""

    def __init__(self, pb):
        self.pb = pb
        self._keep = []
        ch = pb.choices
        a = lambda t, v: self._k(_arr(t, v))  # noqa: E731
        risk = getattr(pb, "evict_risk_permille", None)
        if risk and (pb.billing != 0 or any(not 0 <= r < 1000 for r in risk)):
            raise ValueError("eviction risk needs RESERVED billing and 0 <= rho < 1000 (R32)")
        self.c = OrProblem(
            S=pb.S, dur_us=a(C.c_uint64, pb.dur_us), llm_us=a(C.c_uint64, pb.llm_us),
            tts_us=a(C.c_uint64, pb.tts_us), overhead_us=pb.overhead_us,
            scene0_static=pb.scene0_static, static_ready_us=pb.static_ready_us,
            n_pools=len(pb.gpus), gpus=a(C.c_uint32, pb.gpus),
            price_mc=a(C.c_uint64, pb.price_mc), fixed_cost_mc=pb.fixed_cost_mc,
            billing=pb.billing, objective=pb.objective, n_levels=len(pb.level_score),
            level_score=a(C.c_uint32, pb.level_score), B=len(pb.radix),
            radix=a(C.c_uint32, pb.radix), first_scene=a(C.c_uint32, pb.first_scene),
            choice_level=a(C.c_uint32, [x[0] for x in ch]),
            choice_k=a(C.c_uint32, [x[1] for x in ch]),
            choice_pool=a(C.c_uint32, [x[2] for x in ch]),
            va_us=a(C.c_uint64, pb.va_us),
            pool_ready_us=a(C.c_uint64, pb.pool_ready_us) if getattr(pb, "pool_ready_us", None) else None,
            evict_risk_permille=a(C.c_uint32, risk) if risk else None,
            vae_us=a(C.c_uint64, pb.vae_us) if getattr(pb, "vae_us", None) else None,
            choice_vae_pool=a(C.c_uint32, [0xFFFFFFFF if x is None else x for x in pb.choice_vae_pool])
            if getattr(pb, "vae_us", None) else None,
            metric=getattr(pb, "metric", 0),
            power_active_w=a(C.c_uint32, pb.power_active_w) if getattr(pb, "metric", 0) else None,
            power_idle_w=a(C.c_uint32, pb.power_idle_w) if getattr(pb, "metric", 0) else None)

    def _k(self, x):
        self._keep.append(x)
        return x

    @property
    def n(self) -> int:
        return lib().or_space_size(C.byref(self.c))

    def fixed_stages(self) -> List[int]:
        out = (C.c_uint64 * self.pb.S)()
        lib().or_fixed_stages(C.byref(self.c), out)
        return list(out)

    def deadlines(self) -> List[int]:
        out = (C.c_uint64 * self.pb.S)()
        lib().or_deadlines(C.byref(self.c), out)
        return list(out)

    def decode(self, index: int) -> List[int]:
        out = (C.c_uint32 * len(self.pb.radix))()
        lib().or_decode(C.byref(self.c), C.c_uint64(index), out)
        return list(out)

    def eval(self, index: int):
        """Full detail of one candidate: (Rec, ready_us[S], pool_end[P], makespan, ttff_eff)."""
        S, P = self.pb.S, len(self.pb.gpus)
        a = (C.c_uint64 * S)()
        dl = (C.c_uint64 * S)()
        lib().or_fixed_stages(C.byref(self.c), a)
        lib().or_deadlines(C.byref(self.c), dl)
        r = OrRecord()
        ready = (C.c_uint64 * S)()
        pend = (C.c_uint64 * P)()
        mk = C.c_uint64()
        te = C.c_uint64()
        lib().or_eval_detail(C.byref(self.c), a, dl, C.c_uint64(index), C.byref(r), ready,
                             pend, C.byref(mk), C.byref(te))
        return _rec(r), list(ready), list(pend), mk.value, te.value

    def records(self, begin: int, end: int):
        """Raw OrRecord array for [begin, end) (numpy-viewable)."""
        n = end - begin
        out = (OrRecord * max(1, n))()
        lib().or_eval_range(C.byref(self.c), C.c_uint64(begin), C.c_uint64(end), out)
        return out

    def record_list(self, begin: int, end: int) -> List[Rec]:
        return [_rec(r) for r in self.records(begin, end)][: end - begin]

    def record_hash(self, index: int, rec: Rec) -> int:
        r = OrRecord(*rec.astuple(), 0)
        return lib().or_record_hash(C.c_uint64(index), C.byref(r))

    def sweep(self, begin: int, end: int, queries, nthreads: Optional[int] = None,
              front_cap: int = 1 << 20):
        """Evaluate [begin,end) -> (winners, front, digest).

        winners: list of (status, index, Rec) per query; status 0 feasible,
        1 closest, -1 empty.  front: sorted list of (index, ttff_eff, cost, Q).
        """
        nthreads = nthreads or os.cpu_count() or 1
        nq = len(queries)
        qs = (OrQuery * max(1, nq))(*[OrQuery(q.slo_startup_us, q.slo_stall_us, q.budget_mc)
                                      for q in queries])
        ws = (OrWinner * max(1, nq))()
        fr = (OrPoint * front_cap)()
        fn = C.c_uint64()
        dg = C.c_uint64()
        rc = lib().or_sweep(C.byref(self.c), C.c_uint64(begin), C.c_uint64(end),
                            C.c_uint32(nthreads), C.c_uint32(nq), qs, ws, fr,
                            C.c_uint64(front_cap), C.byref(fn), C.byref(dg))
        if rc != 0:
            raise RuntimeError("or_sweep failed rc=%d (front %d)" % (rc, fn.value))
        winners = [(w.status, w.index, _rec(w.rec)) for w in ws[:nq]]
        front = [(p.index, p.ttff_eff_us, p.cost_mc, p.quality) for p in fr[: fn.value]]
        return winners, front, dg.value


def greedy(orc, query, start=None):
    """Greedy + iterative refinement planner (R28) on the oracle:
    -> (status, index, Rec, iterations, evaluations); status 0 feasible, 1 closest."""
    q = OrQuery(query.slo_startup_us, query.slo_stall_us, query.budget_mc)
    idx = C.c_uint64()
    rec = OrRecord()
    st = C.c_int32()
    it = C.c_uint32()
    ev = C.c_uint64()
    lib().or_greedy(C.byref(orc.c), C.byref(q), C.c_uint64((1 << 64) - 1 if start is None else start),
                    C.byref(idx), C.byref(rec), C.byref(st), C.byref(it), C.byref(ev))
    return st.value, idx.value, _rec(rec), it.value, ev.value


def pareto_points(points):
    """Plain O(n^2) Pareto front of explicit (index, ttff_eff, cost, Q) tuples."""
    n = len(points)
    arr = (OrPoint * max(1, n))(*[OrPoint(i, t, c, q, 0) for (i, t, c, q) in points])
    out = (OrPoint * max(1, n))()
    m = lib().or_pareto_points(arr, C.c_uint64(n), out)
    return [(p.index, p.ttff_eff_us, p.cost_mc, p.quality) for p in out[:m]]


def winner_merge(objective, query, a, b):
    """Merge two (status, index, Rec) winners of one query over disjoint candidate sets
    with the rule or_sweep applies across its threads (or_winner_merge)."""
    q = OrQuery(query.slo_startup_us, query.slo_stall_us, query.budget_mc)

    def w(x):
        st, idx, rec = x
        return OrWinner(idx, OrRecord(*rec.astuple(), 0), st, 0)
    wa, wb, out = w(a), w(b), OrWinner()
    lib().or_winner_merge(C.c_uint32(objective), C.byref(q), C.byref(wa), C.byref(wb), C.byref(out))
    return out.status, out.index, _rec(out.rec)


class OrShared(C.Structure):
    _fields_ = [("n_req", C.c_uint32), ("req", C.POINTER(OrProblem)), ("arrival_us", U64P),
                ("slo_startup_us", U64P), ("slo_stall_us", U64P), ("fixed_index", U64P),
                ("n_pools", C.c_uint32), ("gpus", U32P), ("price_mc", U64P), ("pool_ready_us", U64P),
                ("billing", C.c_uint32), ("objective", C.c_uint32)]


class SharedOracle:
    """Shared-pool fleet (reading R36) of a swgen.SharedFleet: joint
    candidates = the plans of its free requests, evaluated by the per-pool online EDF
    event simulation of or_shared_eval."""

    def __init__(self, sf):
        self.sf = sf
        self.reqs = [Oracle(pb) for pb in sf.requests]
        R = len(self.reqs)
        arr = (OrProblem * R)(*[o.c for o in self.reqs])
        self._keep = [arr]
        a = lambda t, v: self._k(_arr(t, v))  # noqa: E731
        self.c = OrShared(
            n_req=R, req=arr, arrival_us=a(C.c_uint64, sf.arrival_us),
            slo_startup_us=a(C.c_uint64, sf.slo_startup_us), slo_stall_us=a(C.c_uint64, sf.slo_stall_us),
            fixed_index=a(C.c_uint64, [(1 << 64) - 1 if x is None else x for x in sf.fixed_index]),
            n_pools=len(sf.gpus), gpus=a(C.c_uint32, sf.gpus), price_mc=a(C.c_uint64, sf.price_mc),
            pool_ready_us=a(C.c_uint64, sf.pool_ready_us) if sf.pool_ready_us else None,
            billing=sf.billing, objective=sf.objective)

    def _k(self, x):
        self._keep.append(x)
        return x

    @property
    def n(self) -> int:
        lib().or_shared_space_size.restype = C.c_uint64
        return lib().or_shared_space_size(C.byref(self.c))

    def decode(self, index: int) -> List[int]:
        out = (C.c_uint64 * len(self.reqs))()
        lib().or_shared_decode(C.byref(self.c), C.c_uint64(index), out)
        return list(out)

    def eval(self, index: int):
        """-> (fleet Rec, [per-request Rec (cost = its fixed cost)], ready_abs[r][s])."""
        R = len(self.reqs)
        f = OrRecord()
        pr = (OrRecord * R)()
        ready = (C.c_uint64 * (64 * R))()
        lib().or_shared_eval(C.byref(self.c), C.c_uint64(index), C.byref(f), pr, ready)
        return _rec(f), [_rec(x) for x in pr], [list(ready[64 * r: 64 * r + pb.S])
                                                 for r, pb in enumerate(self.sf.requests)]

    def sweep(self, begin: int, end: int, queries, nthreads: Optional[int] = None, front_cap: int = 1 << 20):
        nthreads = nthreads or os.cpu_count() or 1
        nq = len(queries)
        qs = (OrQuery * max(1, nq))(*[OrQuery(q.slo_startup_us, q.slo_stall_us, q.budget_mc) for q in queries])
        ws = (OrWinner * max(1, nq))()
        fr = (OrPoint * front_cap)()
        fn, dg = C.c_uint64(), C.c_uint64()
        rc = lib().or_shared_sweep(C.byref(self.c), C.c_uint64(begin), C.c_uint64(end), C.c_uint32(nthreads),
                                   C.c_uint32(nq), qs, ws, fr, C.c_uint64(front_cap), C.byref(fn), C.byref(dg))
        if rc != 0:
            raise RuntimeError("or_shared_sweep failed rc=%d" % rc)
        return ([(w.status, w.index, _rec(w.rec)) for w in ws[:nq]],
                [(p.index, p.ttff_eff_us, p.cost_mc, p.quality) for p in fr[: fn.value]], dg.value)
