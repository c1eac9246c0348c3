"""Reproduce a random stream parity case and print got vs expected per query (debugging)."""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw  # noqa: E402
from oracle import oracle as orc_mod  # noqa: E402
from swgen import INF  # noqa: E402
from swgen.generator import Query  # noqa: E402
from tests.helpers import random_problem  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
rng = random.Random(500 + seed)
pb = random_problem(rng, max_scenes=7, max_pools=3, max_choices=6, one_scene_digits=rng.random() < 0.5)
pb.queries = [Query(INF, INF, INF), Query(rng.randint(0, 10**8), rng.randint(0, 10**8), rng.randint(0, 10**6)),
              Query(INF, 0, INF), Query(0, 0, 0), Query(INF, INF, rng.randint(0, 10**6))]
o = orc_mod.Oracle(pb)
with sw.Plan(pb, record_capacity=1024) as plan:
    n = plan.n
    w, f, _ = o.sweep(0, n, pb.queries)
    got = plan.stream(0, n, pb.queries)
    for q, (s, (st, i, r)) in enumerate(zip(got, w)):
        print(q, pb.queries[q], "got", s.status, s.index, tuple(s.rec), "exp", st, i, r.astuple())
    print("n", n, "front ok", plan.pareto() == f)
