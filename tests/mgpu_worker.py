"""Multi-GPU parity worker (one rank per GPU, launched by torchrun from
tests/test_gpu_multirank.py): sharded eval (and the sharded fused stream) + NCCL
allgather merge through the C ABI,
compared bit-exactly with the oracle's golden results (tests/golden/, written by
tools/gen_golden.py from oracle/ only)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2603_05800_b200 as sw
    from swgen import make_config
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [sw.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = sw.comm_init(obj[0], rank, world, local)
    cfgs = sys.argv[1:] or ["C3", "C2"]
    for cfg in cfgs:
        pb = make_config(cfg)
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_%s.json" % cfg)))
        n = sw.space_shape(pb)[0]
        if n * 32 > 0.5 * torch.cuda.mem_get_info(local)[0] * world:  # C5: the chunked sweep
            sw.trim_device_memory(local)
            cap = torch.tensor([int(0.75 * torch.cuda.mem_get_info(local)[0]) // 32], device="cuda")
            dist.all_reduce(cap, op=dist.ReduceOp.MIN)  # the sweep is collective: one chunking on every rank
            cap = int(cap.item())
            with sw.Plan(pb, device=local, comm=comm, rank=rank, nranks=world, record_capacity=cap) as plan:
                sels, dg = plan.sweep(0, plan.n, pb.queries, digest=True)
                front = plan.pareto()
        else:
            with sw.Plan(pb, device=local, comm=comm, rank=rank, nranks=world) as plan:
                # global range in two ragged calls: each rank shards both internally
                cut = plan.n // 3 + 12345
                plan.eval(cut, plan.n)
                plan.eval(0, cut)
                sels = plan.select_batch(pb.queries)
                front = plan.pareto()
                dg = plan.digest()
        for s, w in zip(sels, g["winners"]):
            st = {0: 0, 1: 1, -1: 3}[w["status"]]
            assert s.status == st, (cfg, rank, s, w)
            assert s.index == w["index"] and tuple(s.rec) == tuple(w["rec"]), (cfg, rank, s, w)
        assert front == [tuple(p) for p in g["front"]], (cfg, rank, len(front), len(g["front"]))
        assert dg == int(g["digest"]), (cfg, rank)
        # the fused stream path (no records): sharded over the ranks, same winners + front
        with sw.Plan(pb, device=local, comm=comm, rank=rank, nranks=world, record_capacity=1024) as plan:
            ss = plan.stream(0, plan.n, pb.queries)
            sf = plan.pareto()
        for s, w in zip(ss, g["winners"]):
            st = {0: 0, 1: 1, -1: 3}[w["status"]]
            assert s.status == st and s.index == w["index"] and tuple(s.rec) == tuple(w["rec"]), (cfg, rank, s, w)
        assert sf == [tuple(p) for p in g["front"]], (cfg, rank, "stream front")
        print("rank %d/%d %s ok: %d winners, front %d, digest %x (stream too)" % (rank, world, cfg, len(sels),
                                                                                 len(front), dg), flush=True)
    sw.comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
