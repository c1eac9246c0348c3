"""One chunk of C5 (eval of 2^28 candidates + select x3 + fold) -- for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw
from swgen import make_config
pb = make_config("C5")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
plan = sw.Plan(pb, record_capacity=n)
for _ in range(3):
    plan.reset(); plan.eval(0, n); plan.select_batch(pb.queries)
print("C5 chunk ok", plan.launch_count())
