"""C5 chunked sweep time vs record capacity (chunk size): the fold's strided pass count per
chunk depends on the chunk size.  usage: python tools/c5_cap.py CAP [CAP ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_05800_b200 as sw  # noqa: E402
from swgen import make_config  # noqa: E402

pb = make_config("C5")
s = torch.cuda.Stream()
for cap in [int(x) for x in sys.argv[1:]]:
    with sw.Plan(pb, record_capacity=cap, stream=s.cuda_stream) as p:
        for it in range(3):
            p.reset()
            l0 = p.launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            p.sweep(0, p.n, pb.queries)
            e1.record(s)
            e1.synchronize()
        print("cap %d: %.1f ms, %d launches" % (cap, e0.elapsed_time(e1), p.launch_count() - l0), flush=True)
