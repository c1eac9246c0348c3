"""Offline experiments on dumped fold-merge inputs (SW_DUMP_MERGE, tools/gpu_round2.sh
"dump:<cfg>"): how many points each candidate merge strategy leaves for the O(m^2) mark.
usage: python tools/merge_experiment.py gpurun_out/dump/g10_C3_3.bin ..."""
import sys

import numpy as np


def load(path):
    raw = open(path, "rb").read()
    fn = int(np.frombuffer(raw[:8], dtype=np.uint64)[0])
    rec = np.frombuffer(raw[8:], dtype=np.dtype([("idx", "<u8"), ("t", "<u8"), ("c", "<u8"), ("q", "<u4"),
                                                 ("pad", "<u4")]))
    return fn, rec


def dominated_by(P, X):
    """mask over X: some point of P dominates it (<= t, <= c, >= q, one strict)."""
    out = np.zeros(len(X), dtype=bool)
    if len(P) == 0:
        return out
    pt, pc, pq = P["t"].astype(np.int64), P["c"].astype(np.int64), P["q"].astype(np.int64)
    pi = P["idx"].astype(np.uint64)
    for s in range(0, len(X), 512):
        x = X[s:s + 512]
        xt, xc, xq = (x["t"].astype(np.int64)[:, None], x["c"].astype(np.int64)[:, None],
                      x["q"].astype(np.int64)[:, None])
        xi = x["idx"].astype(np.uint64)[:, None]
        le = (pt[None] <= xt) & (pc[None] <= xc) & (pq[None] >= xq)
        st = (pt[None] < xt) | (pc[None] < xc) | (pq[None] > xq) | (pi[None] < xi)  # ties: lowest index
        out[s:s + 512] = (le & st).any(1)
    return out


def local_nd(X, chunk):
    keep = np.zeros(len(X), dtype=bool)
    for s in range(0, len(X), chunk):
        c = X[s:s + chunk]
        keep[s:s + chunk] = ~dominated_by(c, c)
    return keep


def main():
    for path in sys.argv[1:]:
        fn, X = load(path)
        F, S = X[:fn], X[fn:]
        nd = ~dominated_by(X, X)
        print("%s: front %d survivors %d -> merged front %d (new from S %d)" % (path, fn, len(S), nd.sum(),
                                                                               nd[fn:].sum()))
        # (a) current: 256-chunks in buffer order
        k = local_nd(X, 256)
        print("  local 256 buffer order: %d kept" % k.sum())
        # (b) 256-chunks in t order
        o = np.argsort(X["t"], kind="stable")
        k = local_nd(X[o], 256)
        print("  local 256 t-sorted:     %d kept" % k.sum())
        k = local_nd(X[o], 2048)
        print("  local 2048 t-sorted:    %d kept" % k.sum())
        # (c) sample front: every r-th survivor, its ND, then filter everything against it
        for r in (4, 16, 64):
            samp = S[::r]
            sf = samp[~dominated_by(samp, samp)]
            rest = ~dominated_by(sf, S)
            print("  sample 1/%d: %d sampled, sample front %d, survivors left %d" % (r, len(samp), len(sf),
                                                                                     rest.sum()))
        # (d) scalarisation champions: argmin of w.(t/T, c/C, -q/Q) over K weights
        T, C, Q = [float(X[f].max() - X[f].min() + 1) for f in ("t", "c", "q")]
        xs = np.stack([X["t"] / T, X["c"] / C, -X["q"] / Q], 1)
        rng = np.random.default_rng(1)
        for K in (64, 256):
            w = rng.dirichlet([1, 1, 1], K)
            ch = np.unique(np.argmin(xs @ w.T, 0))
            rest = ~dominated_by(X[ch], S)
            print("  champions K=%d: %d distinct, survivors left %d" % (K, len(ch), rest.sum()))


if __name__ == "__main__":
    main()
