"""Full-space oracle result of a large config (C5: 1.2e10 plans), computed in resumable
pieces and cached by the problem's input SHA-256.

Calls ONLY oracle/ (and swgen/ for the seeded inputs); no value comes from the CUDA path.
Each piece [b, e) is one or_sweep (winners, front, digest) written to
tools/.golden_cache/<sha>/piece_<k>.json; when every piece exists the pieces are merged
with the oracle's own rules -- winners by or_winner_merge (the merge or_sweep applies
across its threads), fronts by or_pareto_points over the union (front(A u B) =
front(front(A) u front(B))), digests by addition mod 2^64 -- and written to
tests/golden/oracle_<cfg>.json.

  nice -n 19 python tools/gen_golden_full.py C5 --pieces 256 --threads 7
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from swgen import make_config  # noqa: E402
from oracle.oracle import Oracle, Rec, winner_merge, pareto_points  # noqa: E402
from tools.gen_golden import problem_hash  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--pieces", type=int, default=256)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    pb = make_config(args.config)
    orc = Oracle(pb)
    n = orc.n
    sha = problem_hash(pb)
    cache = os.path.join(ROOT, "tools", ".golden_cache", sha)
    os.makedirs(cache, exist_ok=True)
    P = args.pieces
    for k in range(P):
        path = os.path.join(cache, "piece_%04d_of_%04d.json" % (k, P))
        if os.path.exists(path):
            continue
        b, e = n * k // P, n * (k + 1) // P
        t0 = time.time()
        w, f, d = orc.sweep(b, e, pb.queries, nthreads=args.threads)
        res = {"begin": b, "end": e, "digest": str(d), "seconds": time.time() - t0,
               "winners": [{"status": st, "index": i, "rec": list(r.astuple())} for st, i, r in w],
               "front": [list(p) for p in f]}
        with open(path + ".tmp", "w") as fh:
            json.dump(res, fh)
        os.replace(path + ".tmp", path)
        print("%s piece %d/%d [%d, %d) %.1f s" % (args.config, k + 1, P, b, e, res["seconds"]), flush=True)
    # merge
    wins = [(-1, 0, Rec(0, 0, 0, 0, 0, 0)) for _ in pb.queries]
    pts, dg, secs = [], 0, 0.0
    for k in range(P):
        r = json.load(open(os.path.join(cache, "piece_%04d_of_%04d.json" % (k, P))))
        for q, (qq, w) in enumerate(zip(pb.queries, r["winners"])):
            wins[q] = winner_merge(pb.objective, qq, wins[q], (w["status"], w["index"], Rec(*w["rec"])))
        pts += [tuple(p) for p in r["front"]]
        pts = pareto_points(pts)
        dg = (dg + int(r["digest"])) % (1 << 64)
        secs += r["seconds"]
    out = {"name": pb.name, "sha256": sha, "n": n, "begin": 0, "end": n, "digest": str(dg),
           "queries": [[q.slo_startup_us, q.slo_stall_us, q.budget_mc] for q in pb.queries],
           "winners": [{"status": st, "index": i, "rec": list(r.astuple())} for st, i, r in wins],
           "front": [list(p) for p in pts], "oracle_seconds": secs, "oracle_threads": args.threads,
           "pieces": P}
    path = os.path.join(ROOT, "tests", "golden", "oracle_%s.json" % args.config)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print("done", path, "front", len(pts), flush=True)


if __name__ == "__main__":
    main()
