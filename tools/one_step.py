"""One bench step (reset, eval, select x3, pareto) on a config -- for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw
from swgen import make_config
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pb = make_config(cfg)
plan = sw.Plan(pb)
for _ in range(steps):
    plan.reset(); plan.eval(0, plan.n); plan.select_batch(pb.queries); f = plan.pareto()
print(cfg, "ok", len(f), plan.launch_count())
