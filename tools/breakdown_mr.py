"""Per-call host timing of bench steps under torchrun (rank 0 prints); run with
SW_TRACE=1 for per-phase device times inside select (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2603_05800_b200 as sw
from swgen import make_config
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
comm = None
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [sw.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = sw.comm_init(obj[0], rank, world, local)
pb = make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
s = torch.cuda.Stream()
plan = sw.Plan(pb, device=local, stream=s.cuda_stream, comm=comm, rank=rank, nranks=world)
for it in range(5):
    torch.cuda.synchronize(); a = time.perf_counter()
    plan.reset(); plan.eval(0, plan.n); torch.cuda.synchronize(); b = time.perf_counter()
    plan.select_batch(pb.queries); c = time.perf_counter()
    plan.pareto(); d = time.perf_counter()
    if rank == 0:
        print("world %d: eval %.3f select %.3f pareto %.3f total %.3f ms" % (
            world, 1e3 * (b - a), 1e3 * (c - b), 1e3 * (d - c), 1e3 * (d - a)), flush=True)
if world > 1:
    dist.destroy_process_group()
