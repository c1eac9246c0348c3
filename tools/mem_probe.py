"""Free device memory around handle create/destroy (diagnostic: does the stream-ordered
pool give memory back before the next mem_get_info?)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_05800_b200 as sw  # noqa: E402
from swgen import make_config, make_fleet  # noqa: E402

g = lambda: torch.cuda.mem_get_info(0)[0] / 1e9  # noqa: E731
print("start free %.1f GB" % g())
fleet = make_fleet()
with sw.Fleet(fleet) as F:
    print("fleet alive %.1f GB" % g())
print("after fleet destroy %.1f GB" % g())
torch.cuda.synchronize()
print("after torch.cuda.synchronize %.1f GB" % g())
pb = make_config("C2")
with sw.Plan(pb) as p:
    print("C2 plan alive %.1f GB" % g())
print("after C2 destroy %.1f GB" % g())
torch.cuda.synchronize()
print("after sync %.1f GB" % g())
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
