"""C5 quarter shards on one GPU (diagnostic of the 4-rank imbalance): eval one quarter of the
space, then a select with the config's queries (or subsets), scan time per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_05800_b200 as sw  # noqa: E402
from swgen import make_config  # noqa: E402

pb = make_config("C5")
n = sw.space_shape(pb)[0]
s = torch.cuda.Stream()
cases = (("q0q1q2", [0, 1, 2]), ("q2 only", [2]), ("q0", [0]), ("q1", [1]))
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0].split()[0] in sys.argv[1:]]
for qi, qsel in cases:
    for r in range(4):
        b, e = sw.shard_range(0, n, sw.space_shape(pb)[1], r, 4)
        with sw.Plan(pb, record_capacity=e - b + 4 * sw.space_shape(pb)[1], stream=s.cuda_stream) as p:
            p.eval(b, e)
            k0 = p.kernel_time(sw.SW_KERNEL_SCAN)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            sels = p.select_batch([pb.queries[i] for i in qsel])
            e1.record(s)
            e1.synchronize()
            k1 = p.kernel_time(sw.SW_KERNEL_SCAN)
            print("%-7s quarter %d: select %.1f ms, scan kernels %.1f ms (%d launches), status %s" % (
                qi, r, e0.elapsed_time(e1), k1[1] - k0[1], k1[0] - k0[0], [x.status for x in sels]), flush=True)
