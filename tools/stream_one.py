"""One fused stream call (for ncu captures; diagnostic).  usage: stream_one.py CFG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw
from swgen import make_config

pb = make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # > 1: later calls without first-launch costs
with sw.Plan(pb, record_capacity=1024) as plan:
    for _ in range(reps):
        plan.reset()
        res = plan.stream(0, plan.n, pb.queries)
    print([(s.status, s.index) for s in res])
