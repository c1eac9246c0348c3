"""One fused stream call (for ncu captures; diagnostic).  usage: stream_one.py CFG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw
from swgen import make_config

pb = make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
with sw.Plan(pb, record_capacity=1024) as plan:
    print([(s.status, s.index) for s in plan.stream(0, plan.n, pb.queries)])
