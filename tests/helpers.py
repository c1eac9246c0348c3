"""Test helpers: hand-built planning problems (no method arithmetic here)."""
from swgen.generator import Problem, Query, INF


def make_problem(dur_us, llm_us, tts_us, gpus, price_mc, radix, first_scene, choices,
                 va_us, overhead_us=0, scene0_static=0, static_ready_us=0,
                 fixed_cost_mc=0, billing=0, objective=0, queries=None,
                 level_score=(250, 500, 750, 1000), name="hand", heads=40):
    S = len(dur_us)
    return Problem(
        name=name, S=S, dur_us=list(dur_us), llm_us=list(llm_us), tts_us=list(tts_us),
        overhead_us=overhead_us, scene0_static=scene0_static,
        static_ready_us=static_ready_us, pool_class=["X"] * len(gpus), gpus=list(gpus),
        price_mc=list(price_mc), fixed_cost_mc=fixed_cost_mc, billing=billing,
        objective=objective, level_score=list(level_score), heads=heads, radix=list(radix),
        first_scene=list(first_scene), choices=[tuple(c) for c in choices],
        va_us=list(va_us), queries=queries or [Query(INF, INF, INF)])


def random_problem(rng, max_scenes=5, max_pools=3, max_g=8, max_choices=4,
                   zero_fixed=False, one_scene_digits=True, t_max=50_000_000):
    """Random small problem: every digit a single scene (or random blocks)."""
    S = rng.randint(1, max_scenes)
    n_pools = rng.randint(1, max_pools)
    gpus = [rng.randint(1, max_g) for _ in range(n_pools)]
    price = [rng.choice([180250, 539500, 565250, 106500]) for _ in range(n_pools)]
    dur = [rng.randint(1, 60_000) * 1000 for _ in range(S)]
    if zero_fixed:
        llm = [0] * S
        tts = [0] * S
    else:
        llm = [rng.randint(0, 10_000_000) for _ in range(S)]
        tts = [rng.randint(0, 3_000_000) for _ in range(S)]
    if one_scene_digits:
        first = list(range(S + 1))
    else:
        cuts = sorted(rng.sample(range(1, S), rng.randint(0, S - 1))) if S > 1 else []
        first = [0] + cuts + [S]
    B = len(first) - 1
    radix, choices, va = [], [], []
    for b in range(B):
        r = rng.randint(1, max_choices)
        radix.append(r)
        chs = []
        for _ in range(r):
            p = rng.randrange(n_pools)
            k = rng.randint(1, gpus[p])
            chs.append((rng.randrange(4), k, p))
        choices.extend(chs)
        for s in range(first[b], first[b + 1]):
            for _ in range(r):
                va.append(rng.randint(1, t_max))
    return make_problem(dur, llm, tts, gpus, price, radix, first, choices, va,
                        overhead_us=0 if zero_fixed else rng.randint(0, 2_000_000),
                        fixed_cost_mc=rng.randint(0, 5000),
                        billing=rng.randrange(2), objective=rng.randrange(2),
                        heads=0)  # 0 = no head-divisibility check: exercise any k


def encode(radix, digits):
    """Horner encoding, MSD first (inverse of the decoder)."""
    i = 0
    for r, d in zip(radix, digits):
        i = i * r + d
    return i
