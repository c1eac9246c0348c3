"""Write full-space oracle results to tests/golden/oracle_<cfg>.json.

Calls ONLY oracle/ (and swgen/ for the seeded inputs).  No value here comes from
the CUDA path.  Usage:  python tools/gen_golden.py C1 C2 C3 [C4] [C5] [--threads T]
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


def sweep_json(pb, threads):
    o = Oracle(pb)
    t0 = time.time()
    winners, front, digest = o.sweep(0, o.n, pb.queries, nthreads=threads)
    dt = time.time() - t0
    return {
        "name": pb.name, "sha256": problem_hash(pb), "n": o.n, "digest": str(digest),
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
        if cfg == "C4":
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
