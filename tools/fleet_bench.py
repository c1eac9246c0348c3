"""Time the C4 fleet (256 requests): per-request handles vs the batched sw_fleet API."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_05800_b200 as sw
from swgen import make_fleet

fleet = make_fleet()
s = torch.cuda.Stream()
with sw.Fleet(fleet, stream=s.cuda_stream) as F:
    N = sum(F.plan(i).n for i in range(F.n))
    qs = [pb.queries[0] for pb in fleet]
    for it in range(4):
        torch.cuda.synchronize()
        a = time.perf_counter()
        F.reset(); F.eval()
        torch.cuda.synchronize()
        b = time.perf_counter()
        F.select(qs)
        c = time.perf_counter()
        print("fleet API C4 %d plans: eval %.1f ms, select %.1f ms, total %.1f ms -> %.3g cand/s" % (
            N, 1e3 * (b - a), 1e3 * (c - b), 1e3 * (c - a), N / (c - a)), flush=True)
    print("kernel eval", F.kernel_time(sw.SW_KERNEL_EVAL), "scan", F.kernel_time(sw.SW_KERNEL_SCAN))
plans = [sw.Plan(pb, stream=s.cuda_stream) for pb in fleet]
for it in range(2):
    torch.cuda.synchronize()
    a = time.perf_counter()
    for p in plans:
        p.reset(); p.eval(0, p.n)
    torch.cuda.synchronize()
    b = time.perf_counter()
    for p, pb in zip(plans, fleet):
        p.select_batch(pb.queries)
    c = time.perf_counter()
    print("per-handle C4 %d plans: eval %.1f ms, select %.1f ms, total %.1f ms -> %.3g cand/s" % (
        N, 1e3 * (b - a), 1e3 * (c - b), 1e3 * (c - a), N / (c - a)), flush=True)
