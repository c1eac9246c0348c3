"""Fused streaming mode (sw_plan_stream) timing on one GPU (diagnostic): candidates/s of
whole stream calls (CUDA events on the handle's stream around each call) and the summed
stream-kernel time.  usage: python tools/stream_bench.py [CFG] [STEPS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_05800_b200 as sw
from swgen import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pb = make_config(cfg)
s = torch.cuda.Stream()
with sw.Plan(pb, stream=s.cuda_stream, record_capacity=1024) as plan:
    n = plan.n
    if cfg == "C5":
        n = min(n, 4_000_000_000)
    for _ in range(3):
        plan.reset()
        sels = plan.stream(0, n, pb.queries)
    l0, ms0, _ = plan.kernel_time(sw.SW_KERNEL_STREAM)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(steps):
        plan.reset()
        e0.record(s)
        plan.stream(0, n, pb.queries)
        e1.record(s)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    l1, ms1, _ = plan.kernel_time(sw.SW_KERNEL_STREAM)
    ms = tot / steps
    print("%s stream: %.3f ms/call  %.3e cand/s  stream kernels %.3f ms/call (%d launches/call)  winners %s"
          % (cfg, ms, n / (ms / 1e3), (ms1 - ms0) / steps, (l1 - l0) // steps,
             [(x.status, x.index) for x in sels]), flush=True)
