"""Seeded synthetic inputs shaped like the paper's workloads.

Nothing here evaluates a plan.  The generator only *draws* inputs:

* scene durations (10-minute podcasts split into ~30 s scenes, "10-minute
  video with 30 seconds per shot"), ms-granular, summing exactly to D;
* fixed-stage times from Table 4: StreamCast 1.2 s front end,
  Gemma 6.6 s to the first scene and 31.8 s total, Kokoro 25.8 s for 600 s;
* V+A stage-time tables calibrated to the characterization prose
  (P:532/543 93 s per 81 frames, P:559-560 66/18 s per video-second,
  P:573 pixels, P:580 steps, P:595-596 USP >5x with VAE unparallelised,
  P:669-671 GPU generations);
* integer prices from Table 3 in milli-cents per GPU-hour;
* the select queries (slo_startup_us, slo_stall_us, budget_mc) of each config.

Every floating-point quantity is rounded exactly once (``llround``) into an
integer microsecond / milli-cent table entry; everything downstream is integer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

INF = (1 << 64) - 1  # "no constraint" for a query field

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64 PRNG with named substreams (SPEC S:534 'named random substreams')."""

    def __init__(self, seed: int, stream: str = ""):
        h = 0xCBF29CE484222325  # FNV-1a 64 of the stream name
        for ch in stream.encode():
            h ^= ch
            h = (h * 0x100000001B3) & MASK64
        self.state = (seed ^ h) & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, a: float, b: float) -> float:
        return a + (b - a) * ((self.next_u64() >> 11) * (1.0 / 9007199254740992.0))

    def below(self, n: int) -> int:
        return self.next_u64() % n


def llround(x: float) -> int:
    """C99 llround for x >= 0: round half away from zero, applied once per entry."""
    assert x >= 0.0
    f = math.floor(x)
    return int(f) + (1 if (x - f) >= 0.5 else 0)


# ---------------------------------------------------------------------------
# Quality ladder (P:1346-1349 three tiers; MED+ = ledger L16) and level factor
# LV = pixels x steps relative to MED 640x400/10 ("4x more pixels ...
# approximately 4x higher latency", "DiT latency increases linearly with
# the denoising steps").  Scores are free parameters (ledger L12).
# ---------------------------------------------------------------------------
LEVELS = {
    #        id  width height steps  LV        score
    "LOW":  (0, 320, 200, 5, 1.0 / 8.0, 250),
    "MED":  (1, 640, 400, 10, 1.0, 500),
    "MEDP": (2, 960, 600, 15, 3.375, 750),
    "HIGH": (3, 1280, 800, 20, 8.0, 1000),
}
LEVEL_SCORE = [250, 500, 750, 1000]
LEVEL_LV = [1.0 / 8.0, 1.0, 3.375, 8.0]

# Upscaled rung (reading R34): generate at MED (640x400, 10 steps), then
# Real-ESRGAN to 1280x800 on the same k GPUs.  Table 4: 2663.4 s for the 600 s
# video on one A100 -> 4.439 s per video-second, frames independent (divides by k).
LEVEL_UP = 4
UP_SCORE = 750
ESRGAN_S_PER_VIDEO_S = 2663.4 / 600.0

# DiT speed-up for k GPUs under USP ("over a 5x reduction" at 8;
# ledger L17), VAE/encode fraction 0.12 not parallelised.
SP = {1: 1.0, 2: 1.9, 4: 3.4, 8: 5.2}

# GPU classes: speed vs A100, Table 3 prices converted
# exactly to milli-cents per GPU-hour ($/server-h * 1e5 / GPUs per server).
GPU_CLASSES = {
    #          speed  reserved_mc spot_mc
    "V100":  (None, 134875, 49625),
    "A100":  (1.0, 180250, 106500),
    "H100":  (1.9, 539500, 402750),
    "H200":  (1.995, 565250, 422000),
    "GB200": (2.9, 1441750, 1076000),
}
# GPU power (reading R38): busy = the TDP of Table 3 ("at the highest frequency,
# average power remains within 10% of the peak"); idle = A100's "63W when idle"
# scaled to the class's TDP ("Other GPU generations show similar trends when
# normalized to their TDP"), rounded to whole watts.
GPU_TDP_W = {"V100": 300, "A100": 400, "H100": 700, "H200": 700, "GB200": 1200}
GPU_IDLE_W = {c: (63 * w + 200) // 400 for c, w in GPU_TDP_W.items()}

HEADS = 40  # Wan attention heads; k in {1,2,4,8} all divide it.

# Characterisation anchors, App. B: intercept and slope of the affine
# frames->seconds model from 66 s/s at 1 frame (62.5 ms) and 18 s/s at 81
# frames: 4.125 s = a + b and 93.0 s = a + 81 b.
VA_INTERCEPT_S = 3.0140625
VA_SLOPE_S = 1.1109375


def n16_frames(dur_ms: int) -> int:
    """round(16 * d) compute frames at Wan's 16 FPS."""
    return (16 * dur_ms + 500) // 1000


def va_seconds(dur_ms: int, level: int, k: int, gpu: str, jitter: float = 1.0) -> float:
    """Un-rounded V+A stage time in seconds (App. B), before llround to microseconds."""
    if level == LEVEL_UP:  # MED generation + Real-ESRGAN upscale (R34)
        return (va_seconds(dur_ms, 1, k, gpu, jitter)
                + ESRGAN_S_PER_VIDEO_S * (dur_ms / 1000.0) / (k * GPU_CLASSES[gpu][0]))
    n16 = n16_frames(dur_ms)
    clips = (n16 + 80) // 81  # 81-frame clips
    base = clips * VA_INTERCEPT_S + n16 * VA_SLOPE_S
    return jitter * base * LEVEL_LV[level] * (0.12 + 0.88 / SP[k]) / GPU_CLASSES[gpu][0]


@dataclass
class Query:
    slo_startup_us: int
    slo_stall_us: int
    budget_mc: int


@dataclass
class Problem:
    """One request's planning inputs, exactly as both the oracle and libsw receive them."""
    name: str
    S: int
    dur_us: List[int]
    llm_us: List[int]
    tts_us: List[int]
    overhead_us: int
    scene0_static: int
    static_ready_us: int
    pool_class: List[str]
    gpus: List[int]
    price_mc: List[int]
    fixed_cost_mc: int
    billing: int          # 0 RESERVED, 1 BUSY (ledger L10)
    objective: int        # 0 QUALITY_FIRST, 1 COST_X_TTFF (ledger L13)
    level_score: List[int]
    heads: int
    radix: List[int]
    first_scene: List[int]          # B+1 block boundaries
    choices: List[Tuple[int, int, int]]  # concatenated (level, k, pool) per digit
    va_us: List[int]                # block-major: digit b, scene s in block, choice c
    queries: List[Query] = field(default_factory=list)
    seed: int = 0
    pool_ready_us: List[int] = field(default_factory=list)  # [] = warm pools (R18); R31
    evict_risk_permille: List[int] = field(default_factory=list)  # [] = no Spot risk; R32
    vae_us: List[int] = field(default_factory=list)  # [] = VAE folded into V+A; R37 (block-major)
    choice_vae_pool: List = field(default_factory=list)  # per choice: VAE pool or None; R37
    metric: int = 0                 # 0 cost (milli-cents), 1 energy (microjoules); R38
    power_active_w: List[int] = field(default_factory=list)  # per pool (metric 1)
    power_idle_w: List[int] = field(default_factory=list)

    @property
    def B(self) -> int:
        return len(self.radix)

    @property
    def n_candidates(self) -> int:
        n = 1
        for r in self.radix:
            n *= r
        return n

    def choice_offset(self, b: int) -> int:
        return sum(self.radix[:b])

    def va_offset(self, b: int) -> int:
        off = 0
        for bb in range(b):
            off += (self.first_scene[bb + 1] - self.first_scene[bb]) * self.radix[bb]
        return off


def split_durations(rng: SplitMix64, total_ms: int, S: int) -> List[int]:
    """w_s ~ U[0.6, 1.4]; ms-granular durations summing exactly to total_ms.

    Largest-remainder apportionment, ties to the lower index.
    """
    w = [rng.uniform(0.6, 1.4) for _ in range(S)]
    sw = sum(w)
    raw = [total_ms * x / sw for x in w]
    fl = [int(math.floor(x)) for x in raw]
    rem = total_ms - sum(fl)
    order = sorted(range(S), key=lambda s: (-(raw[s] - fl[s]), s))
    for s in order[:rem]:
        fl[s] += 1
    assert sum(fl) == total_ms and min(fl) > 0
    return fl


def _fixed_stage_times(dur_ms: List[int], scene0_static: bool):
    """Gemma + Kokoro stage times per scene (Table 4; ledger L2/L3)."""
    S = len(dur_ms)
    s0 = 1 if scene0_static else 0
    later = sum(dur_ms[s0 + 1:])
    llm = [0] * S
    tts = [0] * S
    for s in range(s0, S):
        if s == s0:
            llm[s] = 6_600_000  # Gemma first output 6.6 s
        else:
            llm[s] = llround(25.2e6 * dur_ms[s] / later)  # remaining 31.8-6.6 s
        tts[s] = llround(43.0 * dur_ms[s])  # Kokoro 25.8 s / 600 s = 43 ms per s
    return llm, tts


def _build(name, seed, total_s, S, blocks, levels, ks, pools, jitter, static0,
           queries_fn, stream_prefix=""):
    rng_d = SplitMix64(seed, stream_prefix + "durations")
    rng_j = SplitMix64(seed, stream_prefix + "jitter")
    dur_ms = split_durations(rng_d, total_s * 1000, S)
    jit = [rng_j.uniform(0.9, 1.1) if jitter else 1.0 for _ in range(S)]
    llm, tts = _fixed_stage_times(dur_ms, static0)
    pool_class = [p[0] for p in pools]
    gpus = [p[1] for p in pools]
    price = [GPU_CLASSES[c][1] for c in pool_class]  # reserved column
    # level-major, then k, then pool (ledger L19)
    choice_list = []
    for lv in levels:
        for k in ks:
            for p in range(len(pools)):
                if k <= gpus[p]:
                    choice_list.append((lv, k, p))
    radix, first, choices, va = [], [], [], []
    for (lo, hi) in blocks:
        first.append(lo)
        radix.append(len(choice_list))
        choices.extend(choice_list)
        for s in range(lo, hi + 1):
            for (lv, k, p) in choice_list:
                t = llround(1e6 * va_seconds(dur_ms[s], lv, k, pool_class[p], jit[s]))
                va.append(max(1, t))
    first.append(blocks[-1][1] + 1)
    assert first[-1] == S
    # Fixed LLM/TTS instance cost: one A100 over the summed fixed-stage time (App. B).
    fixed_span = 1_200_000 + sum(llm) + sum(tts)
    fixed_cost = llround(GPU_CLASSES["A100"][1] * fixed_span / 3.6e9)
    pb = Problem(
        name=name, S=S, dur_us=[d * 1000 for d in dur_ms], llm_us=llm, tts_us=tts,
        overhead_us=1_200_000, scene0_static=1 if static0 else 0,
        static_ready_us=500_000 if static0 else 0,
        pool_class=pool_class, gpus=gpus, price_mc=price, fixed_cost_mc=fixed_cost,
        billing=0, objective=0, level_score=list(LEVEL_SCORE), heads=HEADS,
        radix=radix, first_scene=first, choices=choices, va_us=va, seed=seed)
    pb.queries = queries_fn(pb)
    return pb


D = 1_000_000  # microseconds per second
DOLLAR = 100_000  # milli-cents per dollar

CONFIG_NAMES = ["C1", "C2", "C3", "C4", "C5"]


def make_config(name: str) -> Problem:
    """The canonical configs of SURVEY §8(d) (BASELINE.json configs[0..4])."""
    if name == "C1":
        # 1-minute podcast, 4 scenes, MED/HIGH, 1 GPU type (A100x2), k in {1,2}: 4^4 = 256.
        return _build("C1", 1001, 60, 4, [(0, 0), (1, 1), (2, 2), (3, 3)],
                      [1, 3], [1, 2], [("A100", 2)], False, False,
                      lambda p: [Query(INF, INF, INF), Query(30 * D, 0, INF),
                                 Query(INF, INF, 342_393)])  # median C1 cost, frozen
    if name == "C2":
        # 10-minute podcast on one 8xA100 server, 20 scenes, 3 levels, k in {1,2,4,8}.
        return _build("C2", 1002, 600, 20,
                      [(0, 0), (1, 1), (2, 2), (3, 3), (4, 8), (9, 13), (14, 18), (19, 19)],
                      [0, 1, 3], [1, 2, 4, 8], [("A100", 8)], True, False,
                      lambda p: [Query(INF, INF, 25 * DOLLAR),      # P:77, "<$25"
                                 Query(120 * D, 0, INF),            # P:1224 "2-minute TTFF"
                                 Query(INF, INF, INF)])
    if name == "C3":
        # Heterogeneous A100+H100, static intro, sub-second startup SLO.
        return _build("C3", 1003, 600, 20,
                      [(1, 1), (2, 2), (3, 3), (4, 11), (12, 18), (19, 19)],
                      [0, 1, 3], [1, 2, 4, 8], [("A100", 8), ("H100", 8)], True, True,
                      lambda p: [Query(999_999, 0, 45 * DOLLAR),    # P:78 "<$45" sub-second
                                 Query(2_999_999, 0, 5 * DOLLAR),   # P:1350 "<3 s"
                                 Query(INF, INF, INF)])
    if name == "C5":
        # 30-minute podcast, 60 scenes, 4 levels x 3 GPU types, 48^6 candidates.
        return _build("C5", 1005, 1800, 60,
                      [(0, 1), (2, 5), (6, 11), (12, 29), (30, 58), (59, 59)],
                      [0, 1, 2, 3], [1, 2, 4, 8],
                      [("A100", 8), ("H100", 8), ("H200", 8)], True, False,
                      lambda p: [Query(60 * D, 0, 150 * DOLLAR),
                                 Query(600 * D, 1800 * D, 100 * DOLLAR),
                                 Query(INF, INF, 40 * DOLLAR)])
    if name == "C2x":
        # C2 under the paper's own objective, "We minimize cost x TTFF" (reading R13:
        # COST_X_TTFF = (cost x ttff_eff as u128, -Q, index)), same space and queries.
        pb = make_config("C2")
        pb.name = "C2x"
        pb.objective = 1
        return pb
    if name == "C3d":
        # C3 with FramePack-style DiT/VAE disaggregation (reading R37): every
        # choice runs its DiT on the chosen pool with k GPUs and streams the latents to a VAE
        # on a separate A100x4 pool (1 GPU per scene; the VAE fraction 0.12 is not
        # parallelised).  Same 24^6 space; t_DiT + t_VAE = C3's V+A time.
        pb = make_config("C3")
        pb.name = "C3d"
        rng_j = SplitMix64(1003, "jitter")
        S = pb.S
        jit = [rng_j.uniform(0.9, 1.1) for _ in range(S)]
        classes = pb.pool_class
        pb.pool_class = classes + ["A100"]
        pb.gpus = pb.gpus + [4]
        pb.price_mc = pb.price_mc + [GPU_CLASSES["A100"][1]]
        va, vae, off = [], [], 0
        for b, r in enumerate(pb.radix):
            chs = pb.choices[sum(pb.radix[:b]): sum(pb.radix[:b]) + r]
            for s in range(pb.first_scene[b], pb.first_scene[b + 1]):
                dms = pb.dur_us[s] // 1000
                n16 = n16_frames(dms)
                base = ((n16 + 80) // 81) * VA_INTERCEPT_S + n16 * VA_SLOPE_S
                for (lv, k, p) in chs:
                    dit = jit[s] * base * LEVEL_LV[lv] * (0.88 / SP[k]) / GPU_CLASSES[classes[p]][0]
                    vs = jit[s] * base * LEVEL_LV[lv] * 0.12 / GPU_CLASSES["A100"][0]
                    va.append(max(1, llround(1e6 * dit)))
                    vae.append(max(1, llround(1e6 * vs)))
        pb.va_us, pb.vae_us = va, vae
        pb.choice_vae_pool = [2] * len(pb.choices)
        return pb
    if name in ("C3e", "C3ex"):
        # C3 scored by ENERGY instead of money ("optimizing for energy ... Energy x
        # TTFF"; reading R38): the record's cost field holds microjoules; budgets are energy
        # budgets.  C3ex minimises Energy x TTFF (the COST_X_TTFF key over energy).
        pb = make_config("C3")
        pb.name = name
        pb.metric = 1
        pb.objective = 1 if name == "C3ex" else 0
        pb.power_active_w = [GPU_TDP_W[c] for c in pb.pool_class]
        pb.power_idle_w = [GPU_IDLE_W[c] for c in pb.pool_class]
        # the LLM/TTS instance: one A100 busy over the fixed-stage span
        fixed_span = pb.overhead_us + sum(pb.llm_us) + sum(pb.tts_us)
        pb.fixed_cost_mc = GPU_TDP_W["A100"] * fixed_span
        MJ = 10 ** 12  # microjoules per megajoule
        pb.queries = [Query(999_999, 0, 4 * MJ), Query(2_999_999, 0, 2 * MJ), Query(INF, INF, INF)]
        return pb
    if name == "C2w":
        # C2 on one 16 x A100 pool ("16xA100"): G_p = 16 > 8 takes the library's
        # generic warp-per-candidate path (SURVEY §8(a) layout note, §8(b) "<= 32 generic").
        return _build("C2w", 1002, 600, 20,
                      [(0, 0), (1, 1), (2, 2), (3, 3), (4, 8), (9, 13), (14, 18), (19, 19)],
                      [0, 1, 3], [1, 2, 4, 8], [("A100", 16)], True, False,
                      lambda p: [Query(INF, INF, 25 * DOLLAR), Query(120 * D, 0, INF), Query(INF, INF, INF)])
    if name == "C3w":
        # C3 with a cold H100 pool: its GPUs are free only after the model load + first
        # warm-up request, 30 s + 80 s (reading R31).
        pb = make_config("C3")
        pb.name = "C3w"
        pb.pool_ready_us = [0, 110 * D]
        return pb
    if name == "C3u":
        # C3 with an upscaled rung: MED + Real-ESRGAN to 1280x800 (P:929-931, P:1196,
        # Table 4, reading R34), scored 750; 32^6 = 1.1e9 plans.
        pb = _build("C3u", 1003, 600, 20,
                    [(1, 1), (2, 2), (3, 3), (4, 11), (12, 18), (19, 19)],
                    [0, 1, LEVEL_UP, 3], [1, 2, 4, 8], [("A100", 8), ("H100", 8)], True, True,
                    lambda p: [Query(999_999, 0, 45 * DOLLAR), Query(2_999_999, 0, 5 * DOLLAR),
                               Query(INF, INF, INF)])
        pb.level_score = LEVEL_SCORE + [UP_SCORE]
        return pb
    if name == "C3t":
        # C3 with a STATIC rung on every digit ("If not enough, we switch to static
        # content", reading R33): choice (STATIC, k = 0)
        # first in each digit's list (quality 0 sorts before LOW, R19), no V+A stage
        # (va_us = 0).  25^6 = 2.4e8 plans.
        pb = make_config("C3")
        pb.name = "C3t"
        static_level = len(pb.level_score)
        pb.level_score = pb.level_score + [0]  # STATIC scores 0 (R12)
        choices, va, off, coff = [], [], 0, 0
        for b, r in enumerate(pb.radix):
            L = pb.first_scene[b + 1] - pb.first_scene[b]
            choices.append((static_level, 0, 0))
            choices.extend(pb.choices[coff:coff + r])
            for j in range(L):
                va.append(0)
                va.extend(pb.va_us[off + j * r: off + (j + 1) * r])
            off += L * r
            coff += r
        pb.radix = [r + 1 for r in pb.radix]
        pb.choices, pb.va_us = choices, va
        return pb
    if name == "C3s":
        # C3 with its H100 pool on Spot VMs: Table 3's Spot column and a 10%
        # eviction risk over the request, covered by over-provisioning (SURVEY
        # §8(f) row 3, reading R32): 8 scheduled H100s are billed as ceil(8 / 0.9) = 9.
        pb = make_config("C3")
        pb.name = "C3s"
        pb.price_mc = [pb.price_mc[0], GPU_CLASSES["H100"][2]]
        pb.evict_risk_permille = [0, 100]
        return pb
    raise KeyError(name)


def make_fleet(n_requests: int = 256, seed: int = 1004) -> List[Problem]:
    """C4: fleet of podcast requests of 5-15 min, per-request SLO/budget (P:1449 mix)."""
    rng = SplitMix64(seed, "fleet")
    out = []
    for r in range(n_requests):
        d_s = 300 + 30 * rng.below(21)
        S = d_s // 30
        h = S // 2
        blocks = [(0, 0), (1, 1), (2, h), (h + 1, S - 2), (S - 1, S - 1)]
        budget = 4 * DOLLAR * d_s // 60  # "$4 per minute" anchors "<$40 per video"
        cls = r % 3

        def qfn(p, cls=cls, budget=budget, d_s=d_s):
            if cls == 0:
                return [Query(30 * D, 0, budget)]                  # real-time
            if cls == 1:
                return [Query(45 * D, d_s * D // 2, budget)]       # relaxed +50%
            return [Query(INF, INF, budget)]                       # batch

        pb = _build("C4.%d" % r, seed, d_s, S, blocks, [0, 1, 3], [1, 2, 4, 8],
                    [("A100", 8), ("H100", 8)], True, False, qfn,
                    stream_prefix="r%d/" % r)
        out.append(pb)
    return out


# ---------------------------------------------------------------------------
# Shared-pool fleets (reading R36): several requests contend for the
# SAME GPU pools, served by per-pool deadline (EDF) queues.  Nothing here
# evaluates a plan: these are the inputs (requests, arrivals, SLOs, background plans).
# ---------------------------------------------------------------------------
@dataclass
class SharedFleet:
    name: str
    requests: List[Problem]        # each request's scenes/tables; choice pools index the shared pools
    arrival_us: List[int]          # T0_r
    slo_startup_us: List[int]      # INF = batch (no SLO)
    slo_stall_us: List[int]
    fixed_index: List               # plan index of a background request, None = free (enumerated)
    gpus: List[int]
    price_mc: List[int]
    pool_ready_us: List[int] = field(default_factory=list)
    billing: int = 0
    objective: int = 0
    queries: List[Query] = field(default_factory=list)

    @property
    def n_candidates(self) -> int:
        n = 1
        for pb, fx in zip(self.requests, self.fixed_index):
            if fx is None:
                n *= pb.n_candidates
        return n


def make_shared(name: str) -> SharedFleet:
    """SF2: two 2-minute requests (4 scenes) planned JOINTLY on shared A100x4 + H100x4
    pools, a real-time one and one arriving 20 s later with a 50%-relaxed SLO.
    SF3: the 1/3 real-time, 1/3 relaxed, 1/3 batch mix: a real-time and a
    batch request in flight (background, fixed plans) and a NEW relaxed 5-minute request
    whose plans are enumerated against that load."""
    pools = [("A100", 4), ("H100", 4)]
    if name == "SF2":
        reqs = []
        for r in range(2):
            pb = _build("SF2.%d" % r, 2001, 120, 4, [(0, 0), (1, 1), (2, 2), (3, 3)], [0, 3], [1, 4],
                        pools, True, False, lambda p: [], stream_prefix="r%d/" % r)
            reqs.append(pb)
        sf = SharedFleet("SF2", reqs, [0, 20 * D], [30 * D, 45 * D], [0, 60 * D], [None, None],
                         [g for _, g in pools], [GPU_CLASSES[c][1] for c, _ in pools])
        sf.queries = [Query(0, 0, INF), Query(0, 0, 40 * DOLLAR), Query(INF, INF, INF)]
        return sf
    if name == "SF3":
        rt = _build("SF3.rt", 2003, 300, 10, [(0, 0), (1, 1), (2, 5), (6, 9)], [0, 1, 3], [1, 2, 4],
                    pools, True, False, lambda p: [], stream_prefix="rt/")
        bt = _build("SF3.batch", 2003, 300, 10, [(0, 0), (1, 1), (2, 5), (6, 9)], [0, 1, 3], [1, 2, 4],
                    pools, True, False, lambda p: [], stream_prefix="batch/")
        new = _build("SF3.new", 2003, 300, 10, [(0, 0), (1, 1), (2, 5), (6, 9)], [0, 1, 3], [1, 2, 4],
                     pools, True, False, lambda p: [], stream_prefix="new/")
        # background plans: real-time at LOW k = 4 on the H100 pool everywhere; batch at
        # MED k = 1 on the A100 pool everywhere (level-major choice order, R19)
        def plan_of(pb, choice):
            c = pb.choices[: pb.radix[0]].index(choice)
            i = 0
            for r in pb.radix:
                i = i * r + c
            return i
        sf = SharedFleet("SF3", [rt, bt, new], [0, 0, 15 * D], [30 * D, INF, 45 * D], [0, INF, 150 * D],
                         [plan_of(rt, (0, 4, 1)), plan_of(bt, (1, 1, 0)), None],
                         [g for _, g in pools], [GPU_CLASSES[c][1] for c, _ in pools])
        sf.queries = [Query(0, 0, INF), Query(0, 0, 30 * DOLLAR), Query(INF, INF, INF)]
        return sf
    raise KeyError(name)
