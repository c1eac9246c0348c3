"""CPU-side checks of the boundary: libsw_plan.so builds, loads without a GPU, exports
every entry point include/sw_plan.h declares; host-only index logic (sharding)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sw():
    from paper_2603_05800_b200 import build
    build.build()
    import paper_2603_05800_b200 as m
    return m


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sw_plan.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sw_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(sw):
    syms = header_symbols()
    assert len(syms) >= 20
    L = ctypes.CDLL(sw.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(sw.EXPORTS), set(syms) ^ set(sw.EXPORTS)
    assert sw.lib().sw_abi_version() == 6 == sw.ABI_VERSION


def test_fails_loudly_without_gpu(sw):
    from tests.conftest import cuda_available
    if cuda_available():
        pytest.skip("GPU present")
    from swgen import make_config
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(make_config("C1"))
    assert ei.value.status == sw.SW_ECUDA


def test_validation_before_device(sw):
    """Input validation happens on the host before any device call."""
    from swgen import make_config
    pb = make_config("C1")
    pb.choices = [(1, 3, 0)] + pb.choices[1:]
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(pb)
    assert ei.value.status == sw.SW_EINVAL
    pb = make_config("C1")
    big = make_config("C5")
    big.va_us = [1 << 61] * len(big.va_us)
    with pytest.raises(sw.SwError) as ei:
        sw.Plan(big)
    assert ei.value.status == sw.SW_ERANGE


@pytest.mark.parametrize("n,row,R", [(10**6 + 7, 144, 8), (144 * 8, 144, 8), (100, 144, 4),
                                     (12**8, 144, 3), (5000, 1, 7)])
def test_shard_range_partitions(sw, n, row, R):
    for begin in (0, 3, 150):
        if begin > n:
            continue
        prev = begin
        for r in range(R):
            b, e = sw.shard_range(begin, n, row, r, R)
            assert b == prev and e >= b
            if 0 < r < R - 1 and e > b:
                assert b % row == 0 and e % row == 0  # interior shards row-aligned
            prev = e
        assert prev == n
