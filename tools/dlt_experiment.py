"""Offline DLT experiments: emulate the device DLT (v5) built from a dumped front on a dumped
record sample and count records that pass it although the front dominates them, for
variants of the binning.  usage: python tools/dlt_experiment.py rec.npy merge_dump.bin"""
import sys

import numpy as np

from merge_experiment import load


def tkey(t, sh=16):
    """float32 bits of t rounded toward zero, >> sh (the device's dlt_tkey: sh = 16)."""
    f = t.astype(np.float64).astype(np.float32)
    over = f.astype(np.float64) > t.astype(np.float64)
    f[over] = np.nextafter(f[over], np.float32(0))
    return (f.view(np.uint32) >> sh).astype(np.int64)


def dlt_pass(F, t, c, q, nt=255, nq=128, t_distinct=False, tmap=False, tsh=16, ncell=2048):
    m = len(F)
    Ft, Fc, Fq = F["t"].astype(np.int64), F["c"].astype(np.int64), F["q"].astype(np.int64)
    if t_distinct:
        dt = np.unique(Ft)
        te = dt if len(dt) <= nt else dt[(np.arange(1, nt + 1) * len(dt)) // nt - 1]
    else:
        te = Ft[(np.arange(nt) * m) // nt]
    dq = np.unique(Fq)
    tops = dq if len(dq) <= nq else dq[(np.arange(1, nq + 1) * len(dq)) // nq - 1]
    cmax = Fc.max()
    csh = 0
    while (cmax >> csh) >= 0xffff:
        csh += 1
    # cell[b][j] = min cost over f with f.t <= te[b] and f.q >= tops[j]
    cell = np.full((len(te) + 1, len(tops) + 1), 0xffff, dtype=np.int64)
    for b in range(len(te)):
        sel = Ft <= te[b]
        for j in range(len(tops)):
            s2 = sel & (Fq >= tops[j])
            if s2.any():
                cell[b + 1, j] = Fc[s2].min() >> csh
    b1 = np.searchsorted(te, t, side="right")
    if tmap:  # the device's 2048-cell direct map: (lo, hi) per cell, hi only if t >= edge[hi-1]
        kbase = tkey(Ft[:1], tsh)[0] - 1
        k = np.clip(tkey(t, tsh) - kbase, 0, ncell - 1)
        ks = np.arange(ncell) + kbase
        def lower_end(kk):
            v = (kk.astype(np.uint32) << tsh).view(np.float32).astype(np.float64)
            return np.ceil(v).astype(np.int64)
        L = lower_end(ks)
        Ln = lower_end(ks + 1)
        U = Ln - 1
        U[-1] = np.iinfo(np.int64).max
        lo = np.searchsorted(te, L, side="right")
        hi = np.searchsorted(te, U, side="right")
        lo_k, hi_k = lo[k], hi[k]
        b1 = np.where((hi_k > lo_k) & (t >= te[np.maximum(hi_k - 1, 0)]), hi_k, lo_k)
        if tmap == "exact":  # a search of the cell's edges when it holds several
            b1 = np.where(hi_k > lo_k + 1, np.searchsorted(te, t, side="right"), b1)
        if tmap == "three":  # branch-free: the cell's first three edges, then its last
            sp = hi_k - lo_k
            tt = lambda i: te[np.minimum(i, len(te) - 1)]
            b1 = lo_k + ((sp >= 1) & (t >= tt(lo_k))) + ((sp >= 2) & (t >= tt(lo_k + 1))) + ((sp >= 3) & (t >= tt(lo_k + 2)))
            b1 = np.where((sp > 3) & (t >= te[np.maximum(hi_k - 1, 0)]), hi_k, b1)
    col = np.searchsorted(tops, q, side="left")
    cs = np.minimum(c >> csh, 0xffff)
    return ~(cs > cell[b1, col])


def exact_dominated(F, t, c, q):
    Ft, Fc, Fq = F["t"].astype(np.int64), F["c"].astype(np.int64), F["q"].astype(np.int64)
    out = np.zeros(len(t), dtype=bool)
    for s in range(0, len(t), 4096):
        tt, cc, qq = t[s:s + 4096, None], c[s:s + 4096, None], q[s:s + 4096, None]
        le = (Ft[None] <= tt) & (Fc[None] <= cc) & (Fq[None] >= qq)
        st = (Ft[None] < tt) | (Fc[None] < cc) | (Fq[None] > qq)
        out[s:s + 4096] = (le & st).any(1)
    return out


def main():
    a = np.load(sys.argv[1])
    fn, X = load(sys.argv[2])
    F = X[:fn]
    t = (a[:, 0] + a[:, 1]).astype(np.int64)
    c = a[:, 2].astype(np.int64)
    q = (a[:, 3] & 0xffffffff).astype(np.int64)
    dom = exact_dominated(F, t, c, q)
    print("records %d, front %d (distinct t %d, q %d); dominated by the front: %d (%.2f%%)" % (
        len(t), fn, len(np.unique(F["t"])), len(np.unique(F["q"])), dom.sum(), 100 * dom.mean()))
    for name, kw in (("v5 255x128", {}), ("v5 + round-1 t map", {"tmap": True}), ("v5 + exact t map", {"tmap": "exact"}), ("v5 + 3-edge t map", {"tmap": "three"}),
                     ("v5 + t map 1/256 oct", {"tmap": True, "tsh": 15, "ncell": 4096}),
                     ("v5 + t map 1/512 oct", {"tmap": True, "tsh": 14, "ncell": 8192}),
                     ("v5 + t map 1/1024 oct", {"tmap": True, "tsh": 13, "ncell": 16384}), ("t distinct 255x128", {"t_distinct": True}),
                     ("255x256", {"nq": 256}), ("t distinct 255x256", {"t_distinct": True, "nq": 256}),
                     ("511x128", {"nt": 511}), ("t distinct 511x64", {"t_distinct": True, "nt": 511, "nq": 64})):
        p = dlt_pass(F, t, c, q, **kw)
        print("  %-22s passes %7d (%.3f%%), of them dominated %7d" % (name, p.sum(), 100 * p.mean(), (p & dom).sum()))


if __name__ == "__main__":
    main()
