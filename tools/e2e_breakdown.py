"""Host-timed breakdown of one end-to-end step through the public API (create from host
tables, sweep, front, destroy) -- where the e2e time beyond the device step goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_05800_b200 as sw  # noqa: E402
from swgen import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
pb = make_config(cfg)
s = torch.cuda.Stream()
N = sw.space_shape(pb)[0]
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = sw.Plan(pb, stream=s.cuda_stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sels, _ = p.sweep(0, N, pb.queries)
    t2 = time.perf_counter()
    f = p.pareto()
    t3 = time.perf_counter()
    p.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print("%s create %.3f sweep %.3f pareto %.3f destroy %.3f total %.3f ms" % (
        cfg, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t4 - t0)))
