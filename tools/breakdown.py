"""Per-call timing of one bench step (diagnostic; runs on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_05800_b200 as sw
from swgen import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
pb = make_config(cfg)
s = torch.cuda.Stream()
plan = sw.Plan(pb, stream=s.cuda_stream)
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    return (time.perf_counter() - a) * 1e3, r
for it in range(3):
    plan.reset()
    te, _ = t(lambda: plan.eval(0, plan.n))
    ts, _ = t(lambda: plan.select_batch(pb.queries))
    ts1, _ = t(lambda: plan.select_batch(pb.queries[:1]))
    tp, f = t(lambda: plan.pareto())
    tp2, f = t(lambda: plan.pareto())
    td, _ = t(lambda: plan.digest())
    print("%s eval %.2f (kernel %.2f) select3 %.2f select1 %.2f pareto %.2f (again %.2f) digest %.2f launches %d front %d" % (
        cfg, te, plan.last_eval_ms(), ts, ts1, tp, tp2, td, plan.launch_count(), len(f)), flush=True)
