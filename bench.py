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
    "C2x": "C2x: C2 under the paper's objective 'We minimize cost x TTFF' (P:918; COST_X_TTFF), 12^8 plans",
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


HBM_SPEC_GBS = 8000.0  # B200 HBM3e spec bandwidth (the measured copy peak is the roofline)


def host_cpu():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "threads": os.cpu_count()}


def load_traffic(cfg):
    """ncu evidence per config (profiles/traffic.json): DRAM bytes / algorithmic bytes and
    issue-active % of one captured launch per kernel."""
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        pj = json.load(open(prof))
    except Exception:
        return {}
    return pj.get("configs", {}).get(cfg, {}).get("kernels", {})


def kernel_roofline(stats0, stats1, steps, ms_per_step, cfg, names=("eval_kernel", "scan_kernel")):
    """Per kernel: ALGORITHMIC bytes per launch (32 B x records written by eval / read by a
    scan) over the launch's CUDA-event time on the handle's stream, averaged over the
    launches of the timed region, against the measured HBM copy peak."""
    peak, peak_kind = peaks()
    tr = load_traffic(cfg)
    kern = {}
    for name, a0, a1 in zip(names, stats0, stats1):
        n_l, t_ms, by = a1[0] - a0[0], a1[1] - a0[1], a1[2] - a0[2]
        if n_l == 0 or t_ms <= 0:
            continue
        avg_ms = t_ms / n_l
        ach = by / n_l / (avg_ms / 1e3) / 1e9
        t = tr.get(name, {})
        kern[name] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                      "pct_of_spec": 100.0 * ach / HBM_SPEC_GBS,
                      "traffic": (t["dram_bytes"] / t["algorithmic_bytes"] * by / n_l) if "dram_bytes" in t else None,
                      "ncu_issue_active_pct": t.get("issue_active_pct"),
                      "algorithmic_bytes_per_launch": by / n_l, "launches": n_l,
                      "ms_per_launch": avg_ms, "share_of_step": t_ms / steps / ms_per_step}
    if not kern:
        return None
    dom = max(kern, key=lambda k: kern[k]["share_of_step"])
    roof = dict(kern[dom])
    roof["kernel"] = dom
    roof["peak_source"] = peak_kind + " (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    roof["kernels"] = kern
    return roof


def measure_plan(ctx, pb, cfg, steps, warmup, e2e_steps, clocks=None):
    """One config through sw_plan_*: STEP = reset + sw_plan_sweep of the whole space (eval,
    records stored, the config's select queries and the Pareto folds; chunked when the
    records exceed 75% of free HBM) + the exact front.  Device time with CUDA events on
    the handle's stream, max over ranks; parity vs the oracle golden after the timed
    region; e2e from host buffers through the public API."""
    import torch
    sw, dev, stream, comm = ctx["sw"], ctx["dev"], ctx["stream"], ctx["comm"]
    rank, world, barrier, mor = ctx["rank"], ctx["world"], ctx["barrier"], ctx["max_over_ranks"]
    N, row = sw.space_shape(pb)
    sw.trim_device_memory(dev)  # earlier configs' handles stay cached in the pool otherwise
    free_b, _ = torch.cuda.mem_get_info(dev)
    need = N // world + 3 * row  # the library's default: this rank's largest shard
    cap_free = int(0.75 * free_b) // REC_BYTES
    if world > 1:  # every rank must chunk the same way (sw_plan_sweep is collective): the min
        cap_free = int(-mor(-float(cap_free)))
    cap = 0 if need < cap_free else cap_free
    out = {"workload": WORKLOADS.get(cfg, cfg), "n_candidates": N, "cap": cap,
           "record_capacity_per_rank": cap, "chunked": cap != 0}

    def step(p):
        p.reset()
        sels, _ = p.sweep(0, N, pb.queries)  # eval (chunked if needed) + select + fold
        return sels, p.pareto()

    plan = sw.Plan(pb, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank, nranks=world,
                   record_capacity=cap)
    for _ in range(warmup):
        step(plan)
    if clocks:
        clocks.start()
        time.sleep(0.3)  # let nvidia-smi start sampling
    barrier()
    l0 = plan.launch_count()
    k0 = [plan.kernel_time(k) for k in (sw.SW_KERNEL_EVAL, sw.SW_KERNEL_SCAN)]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    ev0.record(stream)
    for _ in range(steps):
        sels, front = step(plan)
    ev1.record(stream)
    ev1.synchronize()
    w1 = time.time()
    barrier()
    out["clocks"] = clocks.stop(w0, w1) if clocks else None
    out["gpu_launches"] = plan.launch_count() - l0
    k1 = [plan.kernel_time(k) for k in (sw.SW_KERNEL_EVAL, sw.SW_KERNEL_SCAN)]
    ms = mor(ev0.elapsed_time(ev1))
    out["steps"] = steps
    out["ms_per_step"] = ms / steps
    out["value"] = N / (out["ms_per_step"] / 1e3)
    out["unit"] = UNIT
    out["roofline"] = kernel_roofline(k0, k1, steps, out["ms_per_step"], cfg)
    out["front"] = front
    out["front_points"] = len(front)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "oracle_%s.json" % cfg)
    if os.path.exists(gpath):
        g = json.load(open(gpath))
        if g.get("begin", 0) == 0 and g.get("end", N) == N:
            plan.reset()
            sels_p, dg = plan.sweep(0, N, pb.queries, digest=True)
            ok_w = all(s.index == w["index"] and tuple(s.rec) == tuple(w["rec"])
                       for s, w in zip(sels_p, g["winners"]))
            ok_f = plan.pareto() == [tuple(p) for p in g["front"]]
            parity = {"digest": dg == int(g["digest"]), "winners": ok_w, "pareto": ok_f,
                      "golden_sha256": g.get("sha256")}
    out["parity"] = parity
    plan.close()
    barrier()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(e2e_steps):
        with sw.Plan(pb, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank,
                     nranks=world, record_capacity=cap) as p2:
            s2, f2 = step(p2)
            d2h = 112 * len(s2) + 32 * len(f2)
    barrier()
    e2e_s = mor((time.perf_counter() - t0) / max(1, e2e_steps))
    out["e2e_s"] = e2e_s
    out["d2h"] = d2h
    out["e2e"] = {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": input_bytes(pb),
                  "d2h_bytes_per_step": d2h, "steps": e2e_steps}
    return out


def measure_fleet(ctx, steps, warmup, e2e_steps):
    """C4 (BASELINE configs[3]): 256 requests of 5-15 min, per-request SLO/budget, through
    sw_fleet_*: STEP = reset + one eval launch over every request's space + one select scan
    with one query per request (+ the winners' detail).  Parity: every request's winner and
    record digest vs the oracle golden."""
    import torch
    from swgen import make_fleet
    sw, dev, stream, comm = ctx["sw"], ctx["dev"], ctx["stream"], ctx["comm"]
    rank, world, barrier, mor = ctx["rank"], ctx["world"], ctx["barrier"], ctx["max_over_ranks"]
    fleet = make_fleet()
    qs = [pb.queries[0] for pb in fleet]
    out = {"workload": "C4: fleet of %d podcasts of 5-15 min, A100x8+H100x8 each, per-request SLO/budget "
                       "(real-time / relaxed / batch by r mod 3, P:1449) (BASELINE configs[3])" % len(fleet)}
    with sw.Fleet(fleet, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank, nranks=world) as F:
        N = sum(F.plan(i).n for i in range(F.n))
        out["n_candidates"] = N

        def step():
            F.reset()
            F.eval()
            return F.select(qs)
        for _ in range(warmup):
            step()
        barrier()
        l0 = F.launch_count()
        k0 = [F.kernel_time(k) for k in (sw.SW_KERNEL_EVAL, sw.SW_KERNEL_SCAN)]
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            sels = step()
        ev1.record(stream)
        ev1.synchronize()
        barrier()
        k1 = [F.kernel_time(k) for k in (sw.SW_KERNEL_EVAL, sw.SW_KERNEL_SCAN)]
        ms = mor(ev0.elapsed_time(ev1)) / steps
        out.update(steps=steps, ms_per_step=ms, value=N / (ms / 1e3), unit=UNIT,
                   gpu_launches=F.launch_count() - l0,
                   roofline=kernel_roofline(k0, k1, steps, ms, "C4"))
        gpath = os.path.join(ROOT, "tests", "golden", "oracle_C4.json")
        if os.path.exists(gpath):
            g = json.load(open(gpath))
            ok_w = all(s.index == gr["winners"][0]["index"] and tuple(s.rec) == tuple(gr["winners"][0]["rec"])
                       for s, gr in zip(sels, g["requests"]))
            ok_d = all(F.plan(i).digest() == int(gr["digest"]) for i, gr in enumerate(g["requests"]))
            out["parity"] = {"winners": ok_w, "digest": ok_d}
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        with sw.Fleet(fleet, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank, nranks=world) as F2:
            F2.eval()
            F2.select(qs)
    barrier()
    e2e_s = mor((time.perf_counter() - t0) / max(1, e2e_steps))
    out["e2e"] = {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": sum(input_bytes(pb) for pb in fleet),
                  "d2h_bytes_per_step": 112 * len(fleet), "steps": e2e_steps}
    return out


def input_bytes(pb):
    return (8 * 3 * pb.S + 8 * len(pb.va_us) + 4 * len(pb.radix) + 4 * len(pb.first_scene)
            + 4 * len(pb.choices) + 4 * len(pb.level_score) + 12 * len(pb.gpus))


def emit(line):
    """Print the ONE JSON line on the real stdout (libraries such as NCCL may print to
    fd 1; main() points fd 1 at stderr for the rest of the run)."""
    _REAL_STDOUT.write(json.dumps(line) + "\n")
    _REAL_STDOUT.flush()


_REAL_STDOUT = sys.stdout


def measure_stream(ctx, pb, g, steps):
    """SURVEY §8(f) row 1, reported beside (not instead of) a config's step: the fused
    stream mode evaluates the same space with NO record store (a7 skipped by design),
    select + Pareto filter in-kernel.  CUDA events on the handle's stream around whole
    calls, max over ranks; parity vs the oracle golden (winners + front) when there is one."""
    import torch
    sw, dev, stream, comm = ctx["sw"], ctx["dev"], ctx["stream"], ctx["comm"]
    rank, world = ctx["rank"], ctx["world"]
    N = sw.space_shape(pb)[0]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with sw.Plan(pb, device=dev, stream=stream.cuda_stream, comm=comm, rank=rank, nranks=world,
                 record_capacity=1024) as p3:
        for _ in range(2 if N < 2e9 else 1):
            p3.reset()
            ss = p3.stream(0, N, pb.queries)
        ctx["barrier"]()
        s0 = p3.kernel_time(sw.SW_KERNEL_STREAM)
        ev0.record(stream)
        for _ in range(steps):
            p3.reset()
            ss = p3.stream(0, N, pb.queries)
        ev1.record(stream)
        ev1.synchronize()
        s1 = p3.kernel_time(sw.SW_KERNEL_STREAM)
        sms = ctx["max_over_ranks"](ev0.elapsed_time(ev1) / steps)
        sparity = None
        if g is not None:
            sparity = (all(s.index == w["index"] and tuple(s.rec) == tuple(w["rec"])
                           for s, w in zip(ss, g["winners"])) and
                       p3.pareto() == [tuple(p) for p in g["front"]])
    return {"value": N / (sms / 1e3), "unit": UNIT, "ms_per_call": sms,
            "stream_kernel_ms_per_call": (s1[1] - s0[1]) / steps,
            "launches_per_call": (s1[0] - s0[0]) / steps,
            "calls": steps, "parity": sparity,
            "note": "sw_plan_stream: no records stored (a7 skipped by design; "
                    "SURVEY 8(f) row 1), not the headline step"}


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
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--configs", default="C2x,C3,C4,C5",
                    help="further configs measured after the headline, reported under 'configs'")
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

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            x = float(t[0])
        return x

    ctx = dict(sw=sw, dev=dev, stream=stream, comm=comm, rank=rank, world=world, barrier=barrier,
               max_over_ranks=max_over_ranks)
    clocks = ClockSampler(dev)
    head = measure_plan(ctx, pb, args.config, args.steps, args.warmup, args.e2e_steps, clocks=clocks)
    ms_per_step, value, N, cap = head["ms_per_step"], head["value"], head["n_candidates"], head["cap"]
    ck, launches, roof, parity, front = head["clocks"], head["gpu_launches"], head["roofline"], head["parity"], head["front"]
    e2e_s = head["e2e_s"]
    d2h = head["d2h"]
    gpath = os.path.join(ROOT, "tests", "golden", "oracle_%s.json" % args.config)
    g = json.load(open(gpath)) if os.path.exists(gpath) else None

    stream_line = measure_stream(ctx, pb, g, args.stream_steps) if args.stream_steps > 0 else None

    # the other configs of BASELINE.json / SURVEY 8(d), each a full step of its own
    # workload with per-kernel roofline, parity vs the oracle golden and e2e
    extra = {}
    for cfg in [c for c in args.configs.split(",") if c and c != args.config]:
        try:
            if cfg == "C4":
                extra[cfg] = measure_fleet(ctx, min(args.steps, 10), 3, args.e2e_steps)
            else:
                pbx = make_config(cfg)
                nx = sw.space_shape(pbx)[0]
                st = 3 if nx > 2e9 else min(args.steps, 20)
                r = measure_plan(ctx, pbx, cfg, st, 3 if nx > 2e9 else args.warmup, 1 if nx > 2e9 else args.e2e_steps)
                for k in ("cap", "front", "e2e_s", "d2h", "clocks"):
                    r.pop(k, None)
                if args.stream_steps > 0:
                    gx = os.path.join(ROOT, "tests", "golden", "oracle_%s.json" % cfg)
                    try:
                        r["stream_mode"] = measure_stream(ctx, pbx, json.load(open(gx)) if os.path.exists(gx) else None,
                                                          2 if nx > 2e9 else args.stream_steps)
                    except Exception as ex:  # noqa: BLE001 -- reported, never hides the record path
                        r["stream_mode"] = {"error": "%s: %s" % (type(ex).__name__, ex)}
                extra[cfg] = r
        except Exception as ex:  # noqa: BLE001 -- reported in the line, never hides the headline
            extra[cfg] = {"error": "%s: %s" % (type(ex).__name__, ex)}

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
            "hbm_spec_gbs": HBM_SPEC_GBS,
            "host_cpu": host_cpu(),
            "cpu_baseline": cpu,
            "e2e": {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": input_bytes(pb),
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": ck,
            "parity": parity,
            "front_points": len(front),
            "stream_mode": stream_line,
            "configs": extra,
        }
        emit(line)
    if comm:
        sw.comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
