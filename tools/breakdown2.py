"""Pareto-only fold timing vs chunk size (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from swgen import make_config
cfg = sys.argv[1]
for chunk in sys.argv[2:]:
    os.environ["SW_PARETO_CHUNK"] = chunk
    os.environ["SW_FUSE_PARETO"] = "0"
    import paper_2603_05800_b200 as sw
    pb = make_config(cfg)
    plan = sw.Plan(pb)
    for it in range(2):
        plan.reset(); plan.eval(0, plan.n); torch.cuda.synchronize()
        a = time.perf_counter(); f = plan.pareto(); b = time.perf_counter()
        s = plan.select_batch(pb.queries); c = time.perf_counter()
    print("%s chunk %s pareto-only %.2f ms  select3-plain %.2f ms front %d" % (cfg, chunk, 1e3*(b-a), 1e3*(c-b), len(f)), flush=True)
    plan.close()
