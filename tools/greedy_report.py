"""Greedy planner vs the exhaustive optimum on the GPU: quality,
cost and time of the greedy plan against the exhaustive winner of the same query
(paper: greedy <100 ms, within 20% of optimal cost)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_05800_b200 as sw
from swgen import make_config

out = []
for cfg in sys.argv[1:] or ["C2", "C3"]:
    pb = make_config(cfg)
    with sw.Plan(pb) as plan:
        plan.eval(0, plan.n)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ex = plan.select_batch(pb.queries)
        t_ex = time.perf_counter() - t0
        for qi, (q, e) in enumerate(zip(pb.queries, ex)):
            plan.greedy(q)  # warm
            t0 = time.perf_counter()
            g, it, ev = plan.greedy(q)
            t_g = time.perf_counter() - t0
            row = {"cfg": cfg, "query": qi, "greedy_status": g.status, "exh_status": e.status,
                   "greedy_Q": g.rec[3], "exh_Q": e.rec[3], "greedy_cost_mc": g.rec[2],
                   "exh_cost_mc": e.rec[2], "greedy_ttff_eff": g.ttff_eff_us, "exh_ttff_eff": e.ttff_eff_us,
                   "same_plan": g.index == e.index, "iterations": it, "evaluations": ev,
                   "greedy_ms": 1e3 * t_g, "exhaustive_select_ms_all_queries": 1e3 * t_ex}
            out.append(row)
            print(json.dumps(row), flush=True)
