import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SW_FUSE_PARETO", "0")
import paper_2603_05800_b200 as sw
from swgen import make_config
pb = make_config(sys.argv[1]); plan = sw.Plan(pb); plan.eval(0, plan.n); f = plan.pareto(); print(len(f))
