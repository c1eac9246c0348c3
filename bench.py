#!/usr/bin/env python
"""Bench: batched what-if evaluation of StreamWise serving plans on B200.

One STEP = one pass of the whole hot path over the workload
BASELINE.json's metric is quoted on (configs[1] = C2: 10-minute podcast on one
8xA100-profile server, 20 scenes, 3 levels, k in {1,2,4,8}; 12^8 = 429,981,696
candidate plans): reset, eval of the full space (records stored), the 3 select
queries (one scan), the exact Pareto front, all through the C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Prints ONE JSON line on rank 0.  The oracle (oracle/) is executed only by the
cpu_baseline leg (rank 0, N=1) and by --impl reference.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "plan candidates evaluated/sec (1/2/4/8 B200) and % HBM roofline vs CPU oracle"
UNIT = "candidates/s"
REC_BYTES = 32  # algorithmic HBM bytes per candidate of the eval kernel (the record)
WORKLOADS = {
    "C1": "C1: 1-minute podcast, 4 scenes, MED/HIGH, A100x2, k{1,2}: 256 plans (BASELINE configs[0])",
    "C2": "C2: 10-minute podcast, one 8xA100-profile server, 20 scenes, 3 levels x k{1,2,4,8}, "
          "12^8 plans (BASELINE configs[1])",
    "C3": "C3: 10-minute podcast, A100x8+H100x8, static intro, early low-res ladder, 24^6 plans "
          "(BASELINE configs[2])",
    "C5": "C5: 30-minute podcast, 60 scenes, 4 levels x A100/H100/H200, 48^6 = 1.2e10 plans, "
          "chunked when records exceed HBM (BASELINE configs[4])",
    "C3w": "C3w: C3 with a cold H100 pool ready at 110 s (load 30 s + warm-up 80 s, P:608-611; "
           "SURVEY 8(f) row 3), 24^6 plans",
    "C3u": "C3u: C3 with an upscaled rung (MED + Real-ESRGAN to 1280x800, P:929-931, Table 4; "
           "SURVEY 8(f) row 3), 32^6 = 1.1e9 plans",
    "C3t": "C3t: C3 with a STATIC rung (no video stage, R_s = a_s; P:997, SURVEY 8(f) row 3) on "
           "every digit, 25^6 plans",
    "C3s": "C3s: C3 with the H100 pool on Spot prices (Table 3) and a 10% eviction risk covered "
           "by over-provisioning (9 billed for 8 scheduled, P:939-943; SURVEY 8(f) row 3), 24^6 plans",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms; stop() keeps the samples
    taken inside [t0, t1] (the timed region, wall clock)."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, t0, t1):
        if not self.proc:
            return None
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 10:
                continue
            try:
                ts = time.mktime(time.strptime(p[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                ts += float("0." + p[0].split(".")[1]) if "." in p[0] else 0.0
            except Exception:
                continue
            rows.append((ts, p))
        os.unlink(self.path)
        inside = [p for ts, p in rows if t0 - 0.06 <= ts <= t1 + 0.06]
        if not inside:  # very short timed region: nearest samples
            inside = [p for ts, p in sorted(rows, key=lambda x: abs(x[0] - (t0 + t1) / 2))[:2]]
        if not inside:
            return None

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[2]) for r in inside) if v is not None]
        mx = [v for v in (num(r[3]) for r in inside) if v is not None]
        reasons = set()
        for r in inside:
            for n, v in zip(self.NAMES, r[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(inside), "samples_total": len(rows)}


def cpu_baseline(pb, queries, target_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded prefix of the space."""
    from oracle.oracle import Oracle
    orc = Oracle(pb)
    th = os.cpu_count() or 1
    n0 = 20000 * th
    t = time.perf_counter()
    orc.sweep(0, n0, queries, nthreads=th)
    dt = max(time.perf_counter() - t, 1e-3)
    n = int(min(orc.n, max(n0, n0 * target_s / dt)))
    t = time.perf_counter()
    orc.sweep(0, n, queries, nthreads=th)
    dt = time.perf_counter() - t
    return {"value": n / dt, "unit": UNIT, "cores": th, "kind": "oracle",
            "sample": "%s candidates [0, %d) of %d, full recompute + %d queries + Pareto + digest, "
                      "%.1f s" % (pb.name, n, orc.n, len(queries), dt)}


def run_reference(args, pb):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.oracle import Oracle
    orc = Oracle(pb)
    th = os.cpu_count() or 1
    per_step = 1_000_000 * max(1, th // 8)  # bounded sample per step
    per_step = min(per_step, orc.n)
    off = 0
    for _ in range(args.warmup):
        orc.sweep(off, off + per_step, pb.queries, nthreads=th)
    times = []
    for k in range(args.steps):
        b = (k * per_step) % max(1, orc.n - per_step)
        t = time.perf_counter()
        orc.sweep(b, b + per_step, pb.queries, nthreads=th)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    v = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": "%s (%d candidates); each step a %d-candidate sample" % (
            pb.name, orc.n, per_step), "n_candidates": orc.n, "parallelism": "cpu threads"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": th, "kind": "oracle",
                         "sample": "%d candidates per step, full recompute + %d queries + Pareto"
                                   " + digest" % (per_step, len(pb.queries))},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def input_bytes(pb):
    return (8 * 3 * pb.S + 8 * len(pb.va_us) + 4 * len(pb.radix) + 4 * len(pb.first_scene)
            + 4 * len(pb.choices) + 4 * len(pb.level_score) + 12 * len(pb.gpus))


def emit(line):
    """Print the ONE JSON line on the real stdout (libraries such as NCCL may print to
    fd 1; main() points fd 1 at stderr for the rest of the run)."""
    _REAL_STDOUT.write(json.dumps(line) + "\n")
    _REAL_STDOUT.flush()


_REAL_STDOUT = sys.stdout


def main():
    global _REAL_STDOUT
    _REAL_STDOUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--stream-steps", type=int, default=5,
                    help="fused stream mode (SURVEY §8(f) row 1) calls timed after the main line (0: skip)")
    args = ap.parse_args()

    from swgen import make_config
    pb = make_config(args.config)
    if args.impl == "reference":
        return run_reference(args, pb)

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = local
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2603_05800_b200 as sw
    if world > 1:
        obj = [sw.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = sw.comm_init(obj[0], rank, world, dev)

    stream = torch.cuda.Stream(device=dev)
    N = sw.space_shape(pb)[0]
    # records retained per rank: this rank's share, or as many as 75% of free HBM holds
    # (C5: 391 GB of records -> chunked sweep)
    free_b, _ = torch.cuda.mem_get_info(dev)
    n_max, row = sw.space_shape(pb)
    need = N // world + 3 * row  # the library's default: this rank's largest shard
    cap = 0 if need * REC_BYTES < 0.75 * free_b else int(0.75 * free_b) // REC_BYTES
    plan = sw.Plan(pb, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank, nranks=world,
                   record_capacity=cap)

    def step(p):
        p.reset()
        sels, _ = p.sweep(0, N, pb.queries)  # eval (chunked if needed) + select + fold
        front = p.pareto()
        return sels, front

    for _ in range(args.warmup):
        step(plan)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)  # let nvidia-smi start sampling
    barrier()
    l0 = plan.launch_count()
    k0 = [plan.kernel_time(k) for k in (sw.SW_KERNEL_EVAL, sw.SW_KERNEL_SCAN)]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        sels, front = step(plan)
    ev1.record(stream)
    ev1.synchronize()
    w1 = time.time()
    barrier()
    ck = clocks.stop(w0, w1)
    launches = plan.launch_count() - l0
    k1 = [plan.kernel_time(k) for k in (sw.SW_KERNEL_EVAL, sw.SW_KERNEL_SCAN)]
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    ms_per_step = ms / args.steps
    value = N / (ms_per_step / 1e3)

    # roofline per kernel: ALGORITHMIC bytes per launch (32 B x records written by eval /
    # read by the fused select+Pareto scan) over the launch's CUDA-event time on the
    # handle's stream, averaged over the launches of the timed region; the dominant
    # kernel (largest share of the step) is the line's "roofline"
    peak, peak_kind = peaks()
    traffic = {}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("config") == args.config:
                # per kernel: DRAM bytes / algorithmic bytes of the captured launch
                traffic = {k: v["dram_bytes"] / v["algorithmic_bytes"]
                           for k, v in pj.get("kernels", {}).items()}
        except Exception:
            pass
    kern = {}
    for name, a0, a1 in zip(("eval_kernel", "scan_kernel"), k0, k1):
        n_l, t_ms, by = a1[0] - a0[0], a1[1] - a0[1], a1[2] - a0[2]
        if n_l == 0:
            continue
        avg_ms = t_ms / n_l
        ach = by / n_l / (avg_ms / 1e3) / 1e9
        kern[name] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                      "frac": ach / peak,
                      "traffic": (traffic[name] * by / n_l) if name in traffic else None,
                      "algorithmic_bytes_per_launch": by / n_l, "launches": n_l,
                      "ms_per_launch": avg_ms, "share_of_step": t_ms / args.steps / ms_per_step}
    dom = max(kern, key=lambda k: kern[k]["share_of_step"])
    roof = dict(kern[dom])
    roof["kernel"] = dom
    roof["peak_source"] = peak_kind + " (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    roof["kernels"] = kern

    # parity check of the timed configuration (outside the timed region)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "oracle_%s.json" % args.config)
    if os.path.exists(gpath):
        g = json.load(open(gpath))
        plan.reset()
        sels_p, dg = plan.sweep(0, N, pb.queries, digest=True)
        ok_w = all(s.index == w["index"] and tuple(s.rec) == tuple(w["rec"])
                   for s, w in zip(sels_p, g["winners"]))
        ok_f = plan.pareto() == [tuple(p) for p in g["front"]]
        parity = {"digest": dg == int(g["digest"]), "winners": ok_w, "pareto": ok_f}

    # e2e: public API from HOST buffers each step (create uploads the tables, results
    # come back to host), wall clock with device sync on both sides, max over ranks
    plan.close()
    barrier()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(args.e2e_steps):
        with sw.Plan(pb, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank,
                     nranks=world, record_capacity=cap) as p2:
            s2, f2 = step(p2)
            d2h = 112 * len(s2) + 32 * len(f2)
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])

    # §8(f) row 1, reported beside (not instead of) the headline: the fused stream mode
    # evaluates the same space with NO record store (a7 skipped by design), select + Pareto
    # filter in-kernel; CUDA events on the stream around whole calls, max over ranks
    stream_line = None
    if args.stream_steps > 0:
        with sw.Plan(pb, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank, nranks=world,
                     record_capacity=1024) as p3:
            for _ in range(2):
                p3.reset()
                ss = p3.stream(0, N, pb.queries)
            barrier()
            s0 = p3.kernel_time(sw.SW_KERNEL_STREAM)
            ev0.record(stream)
            for _ in range(args.stream_steps):
                p3.reset()
                ss = p3.stream(0, N, pb.queries)
            ev1.record(stream)
            ev1.synchronize()
            s1 = p3.kernel_time(sw.SW_KERNEL_STREAM)
            sms = ev0.elapsed_time(ev1) / args.stream_steps
            if world > 1:
                t = torch.tensor([sms], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                sms = float(t[0])
            sparity = None
            if os.path.exists(gpath):
                sparity = (all(s.index == w["index"] and tuple(s.rec) == tuple(w["rec"])
                               for s, w in zip(ss, g["winners"])) and
                           p3.pareto() == [tuple(p) for p in g["front"]])
            stream_line = {"value": N / (sms / 1e3), "unit": UNIT, "ms_per_call": sms,
                           "stream_kernel_ms_per_call": (s1[1] - s0[1]) / args.stream_steps,
                           "launches_per_call": (s1[0] - s0[0]) / args.stream_steps,
                           "calls": args.stream_steps, "parity": sparity,
                           "note": "sw_plan_stream: no records stored (a7 skipped by design; "
                                   "SURVEY 8(f) row 1), not the headline step"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(pb, pb.queries)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config),
                       "n_candidates": N, "queries": len(pb.queries),
                       "l2": "records %.1f GB >> 126 MB L2 (no flush needed)" % (N * 32 / 1e9),
                       "record_capacity_per_rank": cap,
                       "parallelism": "candidate-shard x%d, NCCL allgather merge" % world},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": input_bytes(pb),
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": ck,
            "parity": parity,
            "front_points": len(front),
            "stream_mode": stream_line,
        }
        emit(line)
    if comm:
        sw.comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
