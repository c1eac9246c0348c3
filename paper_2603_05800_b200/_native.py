"""Thin ctypes binding of libsw_plan.so (include/sw_plan.h): argument marshalling only.

Every step of the method runs in the library's CUDA kernels.  If the shared library
is missing or no CUDA device is present, calls fail loudly (SwError) -- there is no
CPU fallback.  This module never imports oracle/ (the CPU checker).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
from dataclasses import dataclass
from typing import List, Optional, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsw_plan.so")
# experiment variants (tools/build_variant.py): a differently compiled library, same ABI
_VARIANT = os.environ.get("SW_LIB_VARIANT")
if _VARIANT:
    LIB_PATH = os.path.join(_PKG, "variants", "libsw_plan_%s.so" % _VARIANT)

SW_OK, SW_CLOSEST, SW_TRUNCATED, SW_EMPTY = 0, 1, 2, 3
SW_EINVAL, SW_ERANGE, SW_ENOMEM, SW_ECUDA, SW_ENCCL, SW_ESTATE = -1, -2, -3, -4, -5, -6
SW_KERNEL_EVAL, SW_KERNEL_SCAN, SW_KERNEL_STREAM = 0, 1, 2
SW_MAX_SCENES, SW_MAX_DIGITS, SW_MAX_CHOICES = 64, 16, 64
SW_MAX_POOLS, SW_MAX_GPUS_PER_POOL, SW_MAX_QUERIES = 4, 32, 8
UINT64_MAX = (1 << 64) - 1

U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)


class sw_scene_list(C.Structure):
    _fields_ = [("n_scenes", C.c_uint32), ("dur_us", U64P), ("llm_us", U64P), ("tts_us", U64P),
                ("overhead_us", C.c_uint64), ("scene0_static", C.c_uint32),
                ("static_ready_us", C.c_uint64)]


class sw_choice(C.Structure):
    _fields_ = [("level", C.c_uint8), ("degree", C.c_uint8), ("pool", C.c_uint8), ("vae", C.c_uint8)]


class sw_profile_tables(C.Structure):
    _fields_ = [("n_digits", C.c_uint32), ("radix", U32P), ("first_scene", U32P),
                ("choices", C.POINTER(sw_choice)), ("va_us", U64P), ("n_levels", C.c_uint32),
                ("level_score", U32P), ("heads", C.c_uint32), ("vae_us", U64P)]


class sw_price_table(C.Structure):
    _fields_ = [("n_pools", C.c_uint32), ("gpus", U32P), ("price_mc_per_gpu_hour", U64P),
                ("fixed_cost_mc", C.c_uint64), ("billing", C.c_uint32), ("objective", C.c_uint32),
                ("pool_ready_us", U64P), ("evict_risk_permille", U32P), ("metric", C.c_uint32),
                ("power_active_w", U32P), ("power_idle_w", U32P)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class sw_runtime(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("nccl_comm", C.c_void_p),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("record_capacity", C.c_uint64),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", C.c_void_p)]


class sw_record(C.Structure):
    _fields_ = [("ttff_us", C.c_uint64), ("stall_us", C.c_uint64), ("cost_mc", C.c_uint64),
                ("quality", C.c_uint32), ("stall_count", C.c_uint16), ("flags", C.c_uint8),
                ("pad", C.c_uint8)]

    def astuple(self):
        return (self.ttff_us, self.stall_us, self.cost_mc, self.quality, self.stall_count,
                self.flags)


class sw_query(C.Structure):
    _fields_ = [("slo_startup_us", C.c_uint64), ("slo_stall_us", C.c_uint64),
                ("budget_mc", C.c_uint64)]


class sw_selection(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_uint32), ("index", C.c_uint64),
                ("rec", sw_record), ("ttff_eff_us", C.c_uint64), ("makespan_us", C.c_uint64),
                ("pool_end_us", C.c_uint64 * SW_MAX_POOLS), ("digit", C.c_uint8 * SW_MAX_DIGITS)]


class sw_pareto_point(C.Structure):
    _fields_ = [("index", C.c_uint64), ("ttff_eff_us", C.c_uint64), ("cost_mc", C.c_uint64),
                ("quality", C.c_uint32), ("pad", C.c_uint32)]


_PP_DTYPE = np.dtype([("index", "<u8"), ("t", "<u8"), ("c", "<u8"), ("q", "<u4"), ("pad", "<u4")])

EXPORTS = {
    # name: (restype, argtypes)
    "sw_plan_create": (C.c_int32, [C.POINTER(sw_profile_tables), C.POINTER(sw_scene_list),
                                   C.POINTER(sw_price_table), C.POINTER(sw_runtime),
                                   C.POINTER(C.c_void_p)]),
    "sw_plan_destroy": (C.c_int32, [C.c_void_p]),
    "sw_plan_reset": (C.c_int32, [C.c_void_p]),
    "sw_plan_release_records": (C.c_int32, [C.c_void_p]),
    "sw_plan_space_size": (C.c_int32, [C.c_void_p, U64P]),
    "sw_plan_eval": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64]),
    "sw_plan_select": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                   C.POINTER(sw_selection)]),
    "sw_plan_select_batch": (C.c_int32, [C.c_void_p, C.c_uint32, C.POINTER(sw_query),
                                         C.POINTER(sw_selection)]),
    "sw_plan_sweep": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                  C.POINTER(sw_query), C.POINTER(sw_selection), U64P]),
    "sw_plan_stream": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                   C.POINTER(sw_query), C.POINTER(sw_selection)]),
    "sw_plan_greedy": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                   C.POINTER(sw_selection), C.POINTER(C.c_uint32), U64P]),
    "sw_pareto_get": (C.c_int32, [C.c_void_p, C.POINTER(sw_pareto_point), C.c_uint64, U64P]),
    "sw_plan_digest": (C.c_int32, [C.c_void_p, U64P]),
    "sw_plan_detail": (C.c_int32, [C.c_void_p, C.c_uint64, C.POINTER(sw_selection), U64P]),
    "sw_plan_records": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p), U64P]),
    "sw_plan_copy_records": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64,
                                         C.POINTER(sw_record)]),
    "sw_space_shape": (C.c_int32, [C.POINTER(sw_profile_tables), U64P, U64P]),
    "sw_selection_merge": (C.c_int32, [C.c_uint32, C.POINTER(sw_query), C.POINTER(sw_selection),
                                       C.POINTER(sw_selection), C.POINTER(sw_selection)]),
    "sw_fleet_create": (C.c_int32, [C.c_uint32, C.POINTER(sw_profile_tables), C.POINTER(sw_scene_list),
                                    C.POINTER(sw_price_table), C.POINTER(sw_runtime),
                                    C.POINTER(C.c_void_p)]),
    "sw_fleet_destroy": (C.c_int32, [C.c_void_p]),
    "sw_fleet_size": (C.c_int32, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "sw_fleet_plan": (C.c_int32, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "sw_fleet_eval": (C.c_int32, [C.c_void_p]),
    "sw_fleet_select": (C.c_int32, [C.c_void_p, C.POINTER(sw_query), C.POINTER(sw_selection)]),
    "sw_fleet_reset": (C.c_int32, [C.c_void_p]),
    "sw_fleet_kernel_time": (C.c_int32, [C.c_void_p, C.c_uint32, U64P, C.POINTER(C.c_double), U64P]),
    "sw_fleet_launch_count": (C.c_uint64, [C.c_void_p]),
    "sw_shard_range": (C.c_int32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32,
                                   U64P, U64P]),
    "sw_plan_row_size": (C.c_int32, [C.c_void_p, U64P]),
    "sw_comm_unique_id": (C.c_int32, [C.c_void_p]),
    "sw_comm_init": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                 C.POINTER(C.c_void_p)]),
    "sw_comm_destroy": (C.c_int32, [C.c_void_p]),
    "sw_trim_device_memory": (C.c_int32, [C.c_int32]),
    "sw_status_str": (C.c_char_p, [C.c_int32]),
    "sw_last_error": (C.c_char_p, [C.c_void_p]),
    "sw_plan_launch_count": (C.c_uint64, [C.c_void_p]),
    "sw_plan_last_eval_ms": (C.c_int32, [C.c_void_p, C.POINTER(C.c_float)]),
    "sw_plan_kernel_time": (C.c_int32, [C.c_void_p, C.c_uint32, U64P, C.POINTER(C.c_double), U64P]),
    "sw_abi_version": (C.c_int32, []),
    "sw_plan_decode": (C.c_int32, [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint8)]),
    "sw_plan_segments": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, U64P]),
    "sw_comm_loopback_create": (C.c_int32, [C.c_int32, C.POINTER(C.c_void_p)]),
    "sw_shared_create": (C.c_int32, [C.c_uint32, C.c_void_p, C.c_void_p, U64P, C.c_void_p,
                                     C.POINTER(sw_price_table), C.POINTER(sw_runtime), C.POINTER(C.c_void_p)]),
    "sw_shared_detail": (C.c_int32, [C.c_void_p, C.c_uint64, C.POINTER(sw_record), U64P]),
}
ABI_VERSION = 6

_lib = None


class SwError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (status_str(status), msg))
        self.status = status


def lib():
    """Load libsw_plan.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libsw_plan.so not built: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (nvcc, sm_100a)")
        from . import build as _build
        if not _VARIANT and _build.needs_build():
            raise ImportError("libsw_plan.so is stale (built from other sources than csrc/ + include/): "
                              "rebuild with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.sw_abi_version() != ABI_VERSION:
            raise ImportError("libsw_plan.so ABI %d, binding expects %d" % (L.sw_abi_version(), ABI_VERSION))
        _lib = L
    return _lib


def status_str(s: int) -> str:
    try:
        return lib().sw_status_str(s).decode()
    except Exception:
        return str(s)


def _check(st: int, h=None):
    if st < 0:
        raise SwError(st, lib().sw_last_error(h).decode(errors="replace"))
    return st


def shard_range(begin: int, end: int, row: int, rank: int, nranks: int):
    b, e = C.c_uint64(), C.c_uint64()
    _check(lib().sw_shard_range(begin, end, row, rank, nranks, C.byref(b), C.byref(e)))
    return b.value, e.value


def space_shape(problem):
    """(N, row) of a problem's plan space without a device (sw_space_shape)."""
    radix = _arr(C.c_uint32, problem.radix)
    tb = sw_profile_tables(len(problem.radix), radix, None, None, None, 0, None, 0, None)
    n, row = C.c_uint64(), C.c_uint64()
    _check(lib().sw_space_shape(C.byref(tb), C.byref(n), C.byref(row)))
    return n.value, row.value


def _sel_struct(s: "Selection") -> sw_selection:
    out = sw_selection()
    out.status, out.index = s.status, s.index
    (out.rec.ttff_us, out.rec.stall_us, out.rec.cost_mc, out.rec.quality, out.rec.stall_count,
     out.rec.flags) = s.rec
    out.ttff_eff_us, out.makespan_us = s.ttff_eff_us, s.makespan_us
    for i, v in enumerate(s.pool_end_us[:SW_MAX_POOLS]):
        out.pool_end_us[i] = v
    for i, v in enumerate(s.digit[:SW_MAX_DIGITS]):
        out.digit[i] = v
    return out


def selection_merge(objective: int, query, a: "Selection", b: "Selection") -> "Selection":
    """The better of two selections of one query over disjoint candidate sets
    (sw_selection_merge, host only): chunked sweeps, independent handles, ranks."""
    q = query if isinstance(query, tuple) else (query.slo_startup_us, query.slo_stall_us,
                                                 query.budget_mc)
    sa, sb, out = _sel_struct(a), _sel_struct(b), sw_selection()
    _check(lib().sw_selection_merge(objective, C.byref(sw_query(*q)), C.byref(sa), C.byref(sb),
                                    C.byref(out)))
    return _sel(out, max(len(a.pool_end_us), len(b.pool_end_us)), max(len(a.digit), len(b.digit)))


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().sw_comm_unique_id(buf))
    return bytes(buf)


def comm_init(uid: bytes, rank: int, nranks: int, device: int) -> int:
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    out = C.c_void_p()
    _check(lib().sw_comm_init(buf, rank, nranks, device, C.byref(out)))
    return out.value


def comm_destroy(comm: int) -> None:
    _check(lib().sw_comm_destroy(C.c_void_p(comm)))


def trim_device_memory(device: int = 0) -> None:
    """Return the device's cached, unused pool memory to the driver (sw_trim_device_memory)."""
    _check(lib().sw_trim_device_memory(int(device)))


def comm_loopback_create(nranks: int) -> List[int]:
    """Test/emulation: an in-process loopback group of nranks ranks (sw_comm_loopback_create);
    pass comms[r] as the comm of rank r's handle, one host thread per rank."""
    arr = (C.c_void_p * nranks)()
    _check(lib().sw_comm_loopback_create(nranks, arr))
    return [arr[r] for r in range(nranks)]


class sw_segment(C.Structure):
    _fields_ = [("global_begin", C.c_uint64), ("global_end", C.c_uint64), ("shard_begin", C.c_uint64),
                ("shard_end", C.c_uint64), ("offset", C.c_uint64), ("tile0", C.c_uint64),
                ("ntiles", C.c_uint64), ("row", C.c_uint64)]


@dataclass
class Selection:
    status: int
    index: int
    rec: tuple
    ttff_eff_us: int
    makespan_us: int
    pool_end_us: List[int]
    digit: List[int]


def _sel(s: sw_selection, n_pools: int, B: int) -> Selection:
    return Selection(s.status, s.index, s.rec.astuple(), s.ttff_eff_us, s.makespan_us,
                     list(s.pool_end_us)[:n_pools], list(s.digit)[:B])


def _arr(t, vals):
    vals = list(vals)
    return (t * max(1, len(vals)))(*vals)


def _marshal(pb, keep):
    """ctypes images of a problem's scene list, profile tables and price table."""
    sc = sw_scene_list(pb.S, _arr(C.c_uint64, pb.dur_us), _arr(C.c_uint64, pb.llm_us),
                       _arr(C.c_uint64, pb.tts_us), pb.overhead_us, pb.scene0_static,
                       pb.static_ready_us)
    vae = getattr(pb, "vae_us", None)
    vpool = getattr(pb, "choice_vae_pool", None) or [None] * len(pb.choices)
    chs = (sw_choice * len(pb.choices))(*[sw_choice(l, kk, p, 0 if v is None else v + 1)
                                          for (l, kk, p), v in zip(pb.choices, vpool)])
    tb = sw_profile_tables(len(pb.radix), _arr(C.c_uint32, pb.radix),
                           _arr(C.c_uint32, pb.first_scene), chs, _arr(C.c_uint64, pb.va_us),
                           len(pb.level_score), _arr(C.c_uint32, pb.level_score), pb.heads,
                           _arr(C.c_uint64, vae) if vae else None)
    ready = getattr(pb, "pool_ready_us", None)
    risk = getattr(pb, "evict_risk_permille", None)
    metric = getattr(pb, "metric", 0)
    pr = sw_price_table(len(pb.gpus), _arr(C.c_uint32, pb.gpus), _arr(C.c_uint64, pb.price_mc),
                        pb.fixed_cost_mc, pb.billing, pb.objective,
                        _arr(C.c_uint64, ready) if ready else None,
                        _arr(C.c_uint32, risk) if risk else None, metric,
                        _arr(C.c_uint32, pb.power_active_w) if metric else None,
                        _arr(C.c_uint32, pb.power_idle_w) if metric else None)
    keep.append((sc, chs, tb, pr))
    return sc, tb, pr


class Plan:
    """One request's plan space on one rank (wraps an sw_plan handle).

    ``problem`` is any object with the attributes of the C structs (duck-typed:
    S, dur_us, llm_us, tts_us, overhead_us, scene0_static, static_ready_us, gpus,
    price_mc, fixed_cost_mc, billing, objective, level_score, heads, radix,
    first_scene, choices [(level, k, pool)], va_us).
    """

    def __init__(self, problem, device: int = 0, stream: Optional[int] = None,
                 comm: Optional[int] = None, rank: int = 0, nranks: int = 1,
                 record_capacity: int = 0):
        L = lib()
        pb = problem
        self._keep = []
        sc, tb, pr = _marshal(pb, self._keep)
        rt = sw_runtime(device, C.c_void_p(stream or 0), C.c_void_p(comm or 0), rank, nranks,
                        record_capacity, ALLOC_FN(0), FREE_FN(0), None)
        self._keep.append(rt)
        h = C.c_void_p()
        st = L.sw_plan_create(C.byref(tb), C.byref(sc), C.byref(pr), C.byref(rt), C.byref(h))
        if st < 0:
            raise SwError(st, L.sw_last_error(None).decode(errors="replace"))
        self._adopt(h, pb, owned=True)

    def _adopt(self, h, pb, owned: bool):
        L = lib()
        self.h = h
        self._owned = owned
        self.n_pools = len(pb.gpus)
        self.B = len(pb.radix)
        self.S = pb.S
        n = C.c_uint64()
        L.sw_plan_space_size(h, C.byref(n))
        self.n = n.value
        r = C.c_uint64()
        L.sw_plan_row_size(h, C.byref(r))
        self.row = r.value

    @classmethod
    def borrowed(cls, h, pb) -> "Plan":
        """Wrap a handle owned elsewhere (a fleet's request): close() does not destroy it."""
        self = cls.__new__(cls)
        self._keep = []
        self._adopt(h, pb, owned=False)
        return self

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            if getattr(self, "_owned", True):
                lib().sw_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, st):
        if st < 0:
            raise SwError(st, lib().sw_last_error(self.h).decode(errors="replace"))
        return st

    # -- API (names follow the C ABI)
    def reset(self):
        self._ck(lib().sw_plan_reset(self.h))

    def release_records(self):
        self._ck(lib().sw_plan_release_records(self.h))

    def eval(self, begin: int = 0, end: Optional[int] = None):
        self._ck(lib().sw_plan_eval(self.h, begin, self.n if end is None else end))

    def select(self, slo_startup_us=UINT64_MAX, slo_stall_us=UINT64_MAX, budget_mc=UINT64_MAX):
        out = sw_selection()
        self._ck(lib().sw_plan_select(self.h, slo_startup_us, slo_stall_us, budget_mc, C.byref(out)))
        return _sel(out, self.n_pools, self.B)

    def select_batch(self, queries: Sequence) -> List[Selection]:
        """queries: objects with slo_startup_us / slo_stall_us / budget_mc, or 3-tuples."""
        res = []
        qs = [q if isinstance(q, tuple) else (q.slo_startup_us, q.slo_stall_us, q.budget_mc)
              for q in queries]
        for i in range(0, len(qs), SW_MAX_QUERIES):
            chunk = qs[i:i + SW_MAX_QUERIES]
            arr = (sw_query * len(chunk))(*[sw_query(*q) for q in chunk])
            out = (sw_selection * len(chunk))()
            self._ck(lib().sw_plan_select_batch(self.h, len(chunk), arr, out))
            res += [_sel(o, self.n_pools, self.B) for o in out]
        return res

    def sweep(self, begin: int, end: int, queries: Sequence = (), chunk: int = 0,
              digest: bool = False):
        """Chunked sweep (sw_plan_sweep): -> (selections, digest or None)."""
        qs = [q if isinstance(q, tuple) else (q.slo_startup_us, q.slo_stall_us, q.budget_mc)
              for q in queries]
        arr = (sw_query * max(1, len(qs)))(*[sw_query(*q) for q in qs])
        out = (sw_selection * max(1, len(qs)))()
        d = C.c_uint64()
        self._ck(lib().sw_plan_sweep(self.h, begin, end, chunk, len(qs), arr, out,
                                     C.byref(d) if digest else None))
        return [_sel(o, self.n_pools, self.B) for o in out[: len(qs)]], (d.value if digest else None)

    def stream(self, begin: int, end: int, queries: Sequence = ()):
        """Fused streaming evaluation without records (sw_plan_stream) -> selections."""
        qs = [q if isinstance(q, tuple) else (q.slo_startup_us, q.slo_stall_us, q.budget_mc)
              for q in queries]
        arr = (sw_query * max(1, len(qs)))(*[sw_query(*q) for q in qs])
        out = (sw_selection * max(1, len(qs)))()
        self._ck(lib().sw_plan_stream(self.h, begin, end, len(qs), arr, out))
        return [_sel(o, self.n_pools, self.B) for o in out[: len(qs)]]

    def greedy(self, query=None, start: Optional[int] = None):
        """Greedy + refinement planner (sw_plan_greedy) -> (Selection, iterations,
        evaluations).  query: object / 3-tuple (None = unconstrained)."""
        q = (UINT64_MAX,) * 3 if query is None else (
            query if isinstance(query, tuple) else (query.slo_startup_us, query.slo_stall_us,
                                                    query.budget_mc))
        out = sw_selection()
        it, ev = C.c_uint32(), C.c_uint64()
        self._ck(lib().sw_plan_greedy(self.h, q[0], q[1], q[2], UINT64_MAX if start is None else start,
                                      C.byref(out), C.byref(it), C.byref(ev)))
        return _sel(out, self.n_pools, self.B), it.value, ev.value

    def pareto(self, cap_hint: int = 4096):
        """The exact front (sw_pareto_get) as (index, ttff_eff_us, cost_mc, quality) tuples:
        one call into a buffer kept by the handle, a second only when the front is larger
        (SW_TRUNCATED gives the size)."""
        n = C.c_uint64()
        buf = getattr(self, "_pbuf", None)
        if buf is None or len(buf) < cap_hint:
            buf = self._pbuf = (sw_pareto_point * max(1, cap_hint))()
        st = self._ck(lib().sw_pareto_get(self.h, buf, len(buf), C.byref(n)))
        if st == SW_TRUNCATED:
            buf = self._pbuf = (sw_pareto_point * max(1, n.value))()
            st = self._ck(lib().sw_pareto_get(self.h, buf, len(buf), C.byref(n)))
        assert st == SW_OK
        a = np.frombuffer(buf, dtype=_PP_DTYPE, count=n.value)
        return list(zip(a["index"].tolist(), a["t"].tolist(), a["c"].tolist(), a["q"].tolist()))

    def digest(self) -> int:
        d = C.c_uint64()
        self._ck(lib().sw_plan_digest(self.h, C.byref(d)))
        return d.value

    def detail(self, index: int):
        out = sw_selection()
        ready = (C.c_uint64 * SW_MAX_SCENES)()
        self._ck(lib().sw_plan_detail(self.h, index, C.byref(out), ready))
        return _sel(out, self.n_pools, self.B), list(ready)[: self.S]

    def copy_records(self, index: int, n: int):
        buf = (sw_record * max(1, n))()
        self._ck(lib().sw_plan_copy_records(self.h, index, n, buf))
        return buf

    def decode(self, index: int) -> List[int]:
        """Digit (choice within its digit) of every scene of candidate `index` (sw_plan_decode)."""
        out = (C.c_uint8 * max(1, self.S))()
        self._ck(lib().sw_plan_decode(self.h, index, out))
        return list(out)[: self.S]

    def segments(self):
        """This rank's segment table (sw_plan_segments) as a list of dicts."""
        n = C.c_uint64()
        self._ck(lib().sw_plan_segments(self.h, None, 0, C.byref(n)))
        buf = (sw_segment * max(1, n.value))()
        self._ck(lib().sw_plan_segments(self.h, buf, n.value, C.byref(n)))
        return [{k: getattr(x, k) for k, _ in sw_segment._fields_} for x in buf[: n.value]]

    def records_view(self):
        p = C.c_void_p()
        n = C.c_uint64()
        self._ck(lib().sw_plan_records(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def launch_count(self) -> int:
        return lib().sw_plan_launch_count(self.h)

    def kernel_time(self, kind: int):
        """(launches, summed CUDA-event ms, algorithmic bytes) of one kernel kind since
        create: SW_KERNEL_EVAL, SW_KERNEL_SCAN or SW_KERNEL_STREAM (sw_plan_kernel_time)."""
        n, ms, by = C.c_uint64(), C.c_double(), C.c_uint64()
        self._ck(lib().sw_plan_kernel_time(self.h, kind, C.byref(n), C.byref(ms), C.byref(by)))
        return n.value, ms.value, by.value

    def last_eval_ms(self) -> float:
        ms = C.c_float()
        self._ck(lib().sw_plan_last_eval_ms(self.h, C.byref(ms)))
        return ms.value


class sw_shared_request(C.Structure):
    _fields_ = [("arrival_us", C.c_uint64), ("slo_startup_us", C.c_uint64), ("slo_stall_us", C.c_uint64),
                ("fixed_index", C.c_uint64)]


class SharedPlan(Plan):
    """A shared-pool fleet (sw_shared_create): requests contending for the same pools under
    per-pool EDF queues; the handle is a Plan over the joint plans of the free requests
    (``sf`` duck-typed like swgen.SharedFleet: requests, arrival_us, slo_startup_us,
    slo_stall_us, fixed_index (None = free), gpus, price_mc, pool_ready_us, billing,
    objective)."""

    def __init__(self, sf, device: int = 0, stream: Optional[int] = None, comm: Optional[int] = None,
                 rank: int = 0, nranks: int = 1, record_capacity: int = 0):
        L = lib()
        self._keep = []
        n = len(sf.requests)
        imgs = [_marshal(pb, self._keep) for pb in sf.requests]
        scs = (sw_scene_list * n)(*[i[0] for i in imgs])
        tbs = (sw_profile_tables * n)(*[i[1] for i in imgs])
        fixed = _arr(C.c_uint64, [pb.fixed_cost_mc for pb in sf.requests])
        reqs = (sw_shared_request * n)(*[sw_shared_request(a, t, s, UINT64_MAX if x is None else x)
                                         for a, t, s, x in zip(sf.arrival_us, sf.slo_startup_us,
                                                               sf.slo_stall_us, sf.fixed_index)])
        ready = getattr(sf, "pool_ready_us", None)
        pools = sw_price_table(len(sf.gpus), _arr(C.c_uint32, sf.gpus), _arr(C.c_uint64, sf.price_mc), 0,
                               sf.billing, sf.objective, _arr(C.c_uint64, ready) if ready else None, None,
                               0, None, None)
        rt = sw_runtime(device, C.c_void_p(stream or 0), C.c_void_p(comm or 0), rank, nranks,
                        record_capacity, ALLOC_FN(0), FREE_FN(0), None)
        self._keep += [scs, tbs, fixed, reqs, pools, rt]
        h = C.c_void_p()
        st = L.sw_shared_create(n, C.cast(tbs, C.c_void_p), C.cast(scs, C.c_void_p), fixed,
                                C.cast(reqs, C.c_void_p), C.byref(pools), C.byref(rt), C.byref(h))
        if st < 0:
            raise SwError(st, L.sw_last_error(None).decode(errors="replace"))
        self.sf = sf
        nd = sum(len(pb.radix) for pb, x in zip(sf.requests, sf.fixed_index) if x is None)

        class _Shape:  # what Plan._adopt reads
            gpus, radix, S = sf.gpus, [0] * nd, min(64, sum(pb.S for pb in sf.requests))
        self._adopt(h, _Shape, owned=True)

    def shared_detail(self, index: int):
        """-> ([per-request (ttff, stall, fixed cost, Q, count, 0)], [[absolute ready times] per request])."""
        n = len(self.sf.requests)
        per = (sw_record * n)()
        tot = sum(pb.S for pb in self.sf.requests)
        ready = (C.c_uint64 * max(1, tot))()
        self._ck(lib().sw_shared_detail(self.h, index, per, ready))
        out, off = [], 0
        for pb in self.sf.requests:
            out.append(list(ready[off: off + pb.S]))
            off += pb.S
        return [x.astuple() for x in per], out


class Fleet:
    """A batch of requests evaluated and selected together (sw_fleet_*): one eval launch
    for every request's space, one select scan with one query per request."""

    def __init__(self, problems, device: int = 0, stream: Optional[int] = None,
                 comm: Optional[int] = None, rank: int = 0, nranks: int = 1,
                 record_capacity: int = 0):
        L = lib()
        self.problems = list(problems)
        n = len(self.problems)
        self._keep = []
        imgs = [_marshal(pb, self._keep) for pb in self.problems]
        scs = (sw_scene_list * n)(*[i[0] for i in imgs])
        tbs = (sw_profile_tables * n)(*[i[1] for i in imgs])
        prs = (sw_price_table * n)(*[i[2] for i in imgs])
        rt = sw_runtime(device, C.c_void_p(stream or 0), C.c_void_p(comm or 0), rank, nranks,
                        record_capacity, ALLOC_FN(0), FREE_FN(0), None)
        self._keep.append((scs, tbs, prs, rt))
        h = C.c_void_p()
        st = L.sw_fleet_create(n, tbs, scs, prs, C.byref(rt), C.byref(h))
        if st < 0:
            raise SwError(st, L.sw_last_error(None).decode(errors="replace"))
        self.h = h
        self.n = n

    def close(self):
        if getattr(self, "h", None):
            lib().sw_fleet_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, st):
        if st < 0:
            raise SwError(st, lib().sw_last_error(None).decode(errors="replace"))
        return st

    def plan(self, i: int) -> Plan:
        p = C.c_void_p()
        self._ck(lib().sw_fleet_plan(self.h, i, C.byref(p)))
        return Plan.borrowed(p, self.problems[i])

    def eval(self):
        self._ck(lib().sw_fleet_eval(self.h))

    def reset(self):
        self._ck(lib().sw_fleet_reset(self.h))

    def select(self, queries: Sequence) -> List[Selection]:
        """queries[i] for request i (objects with slo_startup_us / slo_stall_us /
        budget_mc, or 3-tuples)."""
        qs = [q if isinstance(q, tuple) else (q.slo_startup_us, q.slo_stall_us, q.budget_mc)
              for q in queries]
        assert len(qs) == self.n
        arr = (sw_query * self.n)(*[sw_query(*q) for q in qs])
        out = (sw_selection * self.n)()
        self._ck(lib().sw_fleet_select(self.h, arr, out))
        return [_sel(o, len(pb.gpus), len(pb.radix)) for o, pb in zip(out, self.problems)]

    def kernel_time(self, kind: int):
        n, ms, by = C.c_uint64(), C.c_double(), C.c_uint64()
        self._ck(lib().sw_fleet_kernel_time(self.h, kind, C.byref(n), C.byref(ms), C.byref(by)))
        return n.value, ms.value, by.value

    def launch_count(self) -> int:
        return lib().sw_fleet_launch_count(self.h)
