"""Upscaled rung: generate at MED (640x400, 10 steps) and upscale to 1280x800 with
Real-ESRGAN ("run Fantasy Talking at 640x400 and then upscale it to 1280x800 using
Real-ESRGAN"; reading R34).  The rung is a per-scene choice whose
V+A time is the MED generation plus the upscale on the same k GPUs, so it runs through the
unchanged recurrence; what is new is the input recipe, pinned here to Table 4 (P:1183:
Real-ESRGAN 2663.4 s on one A100 for the 10-minute video), and the GPU parity of config C3u
(32^6 plans) against the oracle.  Expected values come only from oracle/ (live) or from
Table 4."""
import random

import pytest

from swgen import make_config
from swgen.generator import va_seconds, LEVEL_UP, GPU_CLASSES
from tests.test_gpu_parity import sw  # noqa: F401 (GPU fixture: skips without CUDA)


def test_upscale_time_reproduces_table4():
    """Summed over the 10-minute C3u podcast (600 s), the upscale part of the rung on one
    A100 (k = 1) is Table 4's 2663.4 s; it divides by k (independent frames) and by the
    GPU speed (H100 1.9x)."""
    pb = make_config("C3u")
    dur_ms = [d // 1000 for d in pb.dur_us]
    assert sum(dur_ms) == 600_000
    up = lambda d, k, g: va_seconds(d, LEVEL_UP, k, g) - va_seconds(d, 1, k, g)  # noqa: E731
    assert abs(sum(up(d, 1, "A100") for d in dur_ms) - 2663.4) < 1e-6
    for d in dur_ms:
        for k in (2, 4, 8):
            assert abs(up(d, k, "A100") - up(d, 1, "A100") / k) < 1e-9
        assert abs(up(d, 1, "H100") - up(d, 1, "A100") / GPU_CLASSES["H100"][0]) < 1e-9


def test_c3u_space():
    """C3u = C3's scenes, pools and queries with the rung between MED and HIGH in the
    level-major choice order (R19): 8 (k, pool) choices per level, 4 levels."""
    a, b = make_config("C3"), make_config("C3u")
    assert b.radix == [32] * 6 and a.radix == [24] * 6
    assert b.level_score[LEVEL_UP] == 750
    assert [c[0] for c in b.choices[:32]] == [0] * 8 + [1] * 8 + [LEVEL_UP] * 8 + [3] * 8
    assert (a.dur_us, a.llm_us, a.tts_us, a.gpus) == (b.dur_us, b.llm_us, b.tts_us, b.gpus)
    # the LOW / MED / HIGH entries are C3's, and each upscaled entry costs more time than
    # MED but less than HIGH for the same (scene, k, pool)
    for s in range(19):
        ra, rb = a.va_us[s * 24:(s + 1) * 24], b.va_us[s * 32:(s + 1) * 32]
        assert rb[:16] == ra[:16] and rb[24:] == ra[16:]
        for j in range(8):
            assert rb[8 + j] < rb[16 + j] < rb[24 + j]


@pytest.mark.gpu
def test_gpu_c3u_subrange(sw, oracle_mod):  # noqa: F811
    """C3u: a ragged 3M sub-range through eval + select + front + digest and the stream
    path; sampled records."""
    from tests.test_gpu_parity import _check_winners, _records_equal
    pb = make_config("C3u")
    orc = oracle_mod.Oracle(pb)
    b, e = 700_000_003, 703_000_041
    w, f, d = orc.sweep(b, e, pb.queries)
    exp = [{"status": st, "index": i, "rec": r.astuple()} for st, i, r in w]
    with sw.Plan(pb, record_capacity=e - b + 10**6) as plan:
        plan.eval(b, e)
        _check_winners(plan.select_batch(pb.queries), exp)
        assert plan.pareto() == f
        assert plan.digest() == d
        rng = random.Random(17)
        for _ in range(20):
            x = rng.randrange(b, e - 256)
            _records_equal(plan, orc, x, x + 256)
    with sw.Plan(pb, record_capacity=1024) as plan:
        _check_winners(plan.stream(b, e, pb.queries), exp)
        assert plan.pareto() == f
