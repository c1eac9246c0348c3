"""Pins of the oracle's DiT/VAE disaggregation (R37) and energy metric (R38); SURVEY §8(f)
row 3, each pinned independently of the oracle's own code.

R37: "FramePack DiT streams latent outputs to the VAE for decoding ... This enables
pipelined execution, independent scaling, and fine-grained resource allocation".
R38: "We also support optimizing for energy, TTFF, and other combinations (e.g., Energy x
TTFF)"; busy GPUs at TDP, idle at 63 W on A100 scaled by TDP.
"""
import random

from swgen import make_config, INF
from swgen.generator import Query, GPU_TDP_W, GPU_IDLE_W, GPU_CLASSES, va_seconds, llround
from tests.helpers import make_problem, random_problem


def _disagg(pb, rng, vae_pool_gpus=None, t_max=20_000_000):
    """Add a VAE pool (last pool) and give every video choice a VAE stage on it."""
    g = vae_pool_gpus or rng.randint(1, 3)
    pb.gpus = pb.gpus + [g]
    pb.price_mc = pb.price_mc + [180250]
    P = len(pb.gpus) - 1
    pb.choice_vae_pool = [P if k > 0 else None for (l, k, p) in pb.choices]
    pb.vae_us = [rng.randint(1, t_max) if v else 0 for v in pb.va_us]
    return P


def _event_sim_2stage(pb, a, digits):
    """Explicit-GPU event simulation, two stages: the DiT takes the k earliest-free GPUs of
    its pool (lowest index on ties), then the VAE the earliest-free GPU of the VAE pool once
    the DiT has finished."""
    free = [[0] * g for g in pb.gpus]
    ready = []
    coff = [sum(pb.radix[:b]) for b in range(pb.B)]
    voff = [pb.va_offset(b) for b in range(pb.B)]
    for s in range(pb.S):
        b = max(bb for bb in range(pb.B) if pb.first_scene[bb] <= s)
        c = digits[b]
        lvl, k, p = pb.choices[coff[b] + c]
        j = voff[b] + (s - pb.first_scene[b]) * pb.radix[b] + c
        t = pb.va_us[j]
        order = sorted(range(pb.gpus[p]), key=lambda gg: (free[p][gg], gg))[:k]
        start = max([a[s]] + [free[p][gg] for gg in order])
        for gg in order:
            free[p][gg] = start + t
        e = start + t
        v = pb.choice_vae_pool[coff[b] + c]
        if v is not None:
            gv = min(range(pb.gpus[v]), key=lambda gg: (free[v][gg], gg))
            sv = max(e, free[v][gv])
            free[v][gv] = sv + pb.vae_us[j]
            e = sv + pb.vae_us[j]
        ready.append(e)
    return ready


def test_disagg_equals_two_stage_event_simulation(oracle_mod):
    rng = random.Random(501)
    for _ in range(1500):
        pb = random_problem(rng, max_scenes=5, max_pools=3)
        _disagg(pb, rng)
        o = oracle_mod.Oracle(pb)
        a = o.fixed_stages()
        i = rng.randrange(o.n)
        rec, ready, pend, mk, te = o.eval(i)
        assert ready == _event_sim_2stage(pb, a, o.decode(i))


def test_disagg_single_scene_closed_form(oracle_mod):
    """One scene, idle pools: R_0 = a_0 + t_DiT + t_VAE; RESERVED cost bills the DiT pool
    (G x R_0... its span ends at a_0 + t_DiT) and the VAE pool (until R_0)."""
    pb = make_problem([30_000_000], [6_600_000], [1_290_000], [8, 1], [180250, 180250], [1], [0, 1],
                      [(3, 2, 0)], [300_000_000], overhead_us=1_200_000, heads=0)
    pb.choice_vae_pool = [1]
    pb.vae_us = [50_000_000]
    rec, ready, pend, mk, te = oracle_mod.Oracle(pb).eval(0)
    a0 = 1_200_000 + 6_600_000 + 1_290_000
    assert ready == [a0 + 300_000_000 + 50_000_000]
    assert pend == [a0 + 300_000_000, a0 + 350_000_000]
    assert rec.cost_mc == (8 * pend[0] * 180250 + 1_800_000_000) // 3_600_000_000 + \
        (1 * pend[1] * 180250 + 1_800_000_000) // 3_600_000_000


def test_disagg_pipelining_never_later(oracle_mod):
    """With a VAE pool that never queues (a GPU per scene), moving the VAE off the DiT
    GPUs only frees them earlier: every scene is ready no later than with the VAE folded
    into the V+A stage on the DiT GPUs (t = t_DiT + t_VAE), and the DiT pool ends no later."""
    rng = random.Random(502)
    for _ in range(800):
        pb = random_problem(rng, max_scenes=5, max_pools=2)
        _disagg(pb, rng, vae_pool_gpus=pb.S)
        o = oracle_mod.Oracle(pb)
        folded = make_problem(pb.dur_us, pb.llm_us, pb.tts_us, pb.gpus, pb.price_mc, pb.radix, pb.first_scene,
                              pb.choices, [t + v for t, v in zip(pb.va_us, pb.vae_us)],
                              overhead_us=pb.overhead_us, heads=0)
        of = oracle_mod.Oracle(folded)
        i = rng.randrange(o.n)
        _, r1, p1, _, _ = o.eval(i)
        _, r2, p2, _, _ = of.eval(i)
        assert all(x <= y for x, y in zip(r1, r2))
        assert all(x <= y for x, y in zip(p1[:-1], p2[:-1]))


def test_c3d_split_preserves_total_time():
    """C3d's split of C3's V+A stage: on the A100 pool t_DiT + t_VAE = C3's V+A time; on the
    H100 pool the VAE moved to an A100 (1.9x slower), so t_DiT + t_VAE / 1.9 =
    C3's V+A time -- up to the roundings (llround once per entry, R24)."""
    c3, c3d = make_config("C3"), make_config("C3d")
    assert len(c3.va_us) == len(c3d.va_us) == len(c3d.vae_us)
    j = 0
    for b, r in enumerate(c3.radix):
        chs = c3.choices[sum(c3.radix[:b]): sum(c3.radix[:b]) + r]
        for s in range(c3.first_scene[b], c3.first_scene[b + 1]):
            for (l, k, p) in chs:
                v, d, e = c3.va_us[j], c3d.va_us[j], c3d.vae_us[j]
                assert abs(v - (d + e / (1.0 if p == 0 else 1.9))) <= 2, (b, s, l, k, p)
                j += 1


# ---- R38: energy ---------------------------------------------------------------------
def test_energy_worked_example(oracle_mod):
    """8 x A100 pool, one scene on k = 1 GPU for one hour after 1 s of fixed stages:
    busy 400 W x 3600 s, the 7 other rented GPUs idle at 63 W for (1 h + 1 s) and the busy
    GPU idle for its first second: E = 400*3.6e9 + 63*(8*(3.6e9 + 1e6) - 3.6e9) uJ."""
    pb = make_problem([60_000_000], [1_000_000], [0], [8], [180250], [1], [0, 1], [(3, 1, 0)], [3_600_000_000],
                      heads=0)
    pb.metric, pb.power_active_w, pb.power_idle_w = 1, [400], [63]
    rec = oracle_mod.Oracle(pb).eval(0)[0]
    assert rec.cost_mc == 400 * 3_600_000_000 + 63 * (8 * 3_601_000_000 - 3_600_000_000)
    pb.billing = 1  # BUSY: busy GPU time only
    assert oracle_mod.Oracle(pb).eval(0)[0].cost_mc == 400 * 3_600_000_000


def test_energy_generation_ratios_match_paper(oracle_mod):
    """"Relative to A100, H100 and H200 reduce total energy consumption by 7% and
    12%, respectively, while GB200 consumes 2% more".  Busy energy of the same scene on one
    GPU of each class (BUSY accounting, TDP x time at the class's speed):
    H100 -7.9%, H200 -12.3%, GB200 +3.4% -- the paper's figures within ~1.5 points."""
    E = {}
    for cls in ("A100", "H100", "H200", "GB200"):
        t = llround(1e6 * va_seconds(30_000, 3, 1, cls))
        pb = make_problem([30_000_000], [0], [0], [1], [GPU_CLASSES[cls][1]], [1], [0, 1], [(3, 1, 0)], [t],
                          billing=1, heads=0)
        pb.metric, pb.power_active_w, pb.power_idle_w = 1, [GPU_TDP_W[cls]], [GPU_IDLE_W[cls]]
        E[cls] = oracle_mod.Oracle(pb).eval(0)[0].cost_mc
    assert abs(E["H100"] / E["A100"] - 0.93) < 0.015
    assert abs(E["H200"] / E["A100"] - 0.88) < 0.015
    assert abs(E["GB200"] / E["A100"] - 1.02) < 0.02


def test_energy_idle_watts():
    """63 W idle on the 400 W A100, other classes scaled by TDP."""
    assert GPU_IDLE_W["A100"] == 63 and GPU_IDLE_W["H100"] == 110 and GPU_IDLE_W["GB200"] == 189


def test_energy_equals_hand_sum_over_event_simulation(oracle_mod):
    """Random problems: the energy record equals sum_p (P_act busy_p + P_idle (G end_p -
    busy_p)) computed by hand from an explicit event simulation's pool ends and busy times."""
    rng = random.Random(503)
    for _ in range(300):
        pb = random_problem(rng, max_scenes=4, max_pools=3)
        pb.metric = 1
        pb.power_active_w = [rng.randint(100, 1200) for _ in pb.gpus]
        pb.power_idle_w = [rng.randint(10, 200) for _ in pb.gpus]
        o = oracle_mod.Oracle(pb)
        i = rng.randrange(o.n)
        rec, ready, pend, mk, te = o.eval(i)
        digs = o.decode(i)
        busy = [0] * len(pb.gpus)
        coff = [sum(pb.radix[:b]) for b in range(pb.B)]
        for s in range(pb.S):
            b = max(bb for bb in range(pb.B) if pb.first_scene[bb] <= s)
            l, k, p = pb.choices[coff[b] + digs[b]]
            busy[p] += k * pb.va_us[pb.va_offset(b) + (s - pb.first_scene[b]) * pb.radix[b] + digs[b]]
        E = pb.fixed_cost_mc
        for p, g in enumerate(pb.gpus):
            if pend[p] == 0:
                continue  # unused pool: not rented
            idle = g * pend[p] - busy[p] if pb.billing == 0 else 0
            E += pb.power_active_w[p] * busy[p] + pb.power_idle_w[p] * idle
        assert rec.cost_mc == E
