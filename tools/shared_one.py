"""One shared-pool fleet pass (eval + select + Pareto) -- diagnostics (SW_DEBUG=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw
from swgen import make_shared
sf = make_shared(sys.argv[1] if len(sys.argv) > 1 else "SF2")
with sw.SharedPlan(sf) as plan:
    plan.eval(0, plan.n)
    print([(s.status, s.index) for s in plan.select_batch(sf.queries)])
    print("front", len(plan.pareto()))
