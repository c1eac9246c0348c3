"""Write full-space oracle results to tests/golden/oracle_<cfg>.json.

Calls ONLY oracle/ (and swgen/ for the seeded inputs).  No value here comes from
the CUDA path.  Usage:  python tools/gen_golden.py C1 C2 C3 [C4] [C5sub] [--threads T]
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from swgen import make_config, make_fleet  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402


def problem_hash(pb) -> str:
    d = {k: v for k, v in sorted(vars(pb).items()) if k not in ("queries", "name")}
    d["queries"] = [[q.slo_startup_us, q.slo_stall_us, q.budget_mc] for q in pb.queries]
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()


# C5 (1.2e10 plans, ~2.2e4 core-s for the full space) is pinned on fixed sub-ranges:
# one from the start of the space and one ragged range in the middle.
C5_RANGES = [(0, 50_000_000), (6_000_000_007, 6_000_000_007 + 20_000_000)]


def sweep_json(pb, threads, begin=0, end=None):
    o = Oracle(pb)
    end = o.n if end is None else end
    t0 = time.time()
    winners, front, digest = o.sweep(begin, end, pb.queries, nthreads=threads)
    dt = time.time() - t0
    return {
        "name": pb.name, "sha256": problem_hash(pb), "n": o.n, "begin": begin, "end": end,
        "digest": str(digest),
        "queries": [[q.slo_startup_us, q.slo_stall_us, q.budget_mc] for q in pb.queries],
        "winners": [{"status": st, "index": idx, "rec": list(r.astuple())}
                    for st, idx, r in winners],
        "front": [list(p) for p in front],
        "oracle_seconds": dt, "oracle_threads": threads,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    out_dir = os.path.join(ROOT, "tests", "golden")
    for cfg in args.configs:
        if cfg == "C5sub":
            pb = make_config("C5")
            res = {"name": "C5sub", "ranges": [sweep_json(pb, args.threads, b, e)
                                               for b, e in C5_RANGES]}
        elif cfg.startswith("SF"):  # shared-pool fleets
            from swgen import make_shared
            from oracle.oracle import SharedOracle
            sf = make_shared(cfg)
            o = SharedOracle(sf)
            t0 = time.time()
            w, f, d = o.sweep(0, o.n, sf.queries, nthreads=args.threads)
            res = {"name": cfg, "n": o.n, "begin": 0, "end": o.n, "digest": str(d),
                   "queries": [[q.slo_startup_us, q.slo_stall_us, q.budget_mc] for q in sf.queries],
                   "winners": [{"status": st, "index": i, "rec": list(r.astuple())} for st, i, r in w],
                   "front": [list(p) for p in f], "oracle_seconds": time.time() - t0,
                   "oracle_threads": args.threads}
        elif cfg == "C4":
            reqs = [sweep_json(pb, args.threads) for pb in make_fleet()]
            res = {"name": "C4", "requests": reqs}
        else:
            res = sweep_json(make_config(cfg), args.threads)
        path = os.path.join(out_dir, "oracle_%s.json" % cfg)
        with open(path, "w") as f:
            json.dump(res, f, indent=0)
        print(cfg, "done", path, flush=True)


if __name__ == "__main__":
    main()
