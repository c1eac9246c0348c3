"""Seeded synthetic workload generator for the StreamWise plan evaluator.

This package is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA product path (``paper_2603_05800_b200/``).  It draws the inputs of a
planning problem (scene durations, fixed-stage times, V+A stage-time tables,
pools, prices, queries) and holds none of the method's arithmetic: no ready
times, no max-plus recurrence, no metrics, no cost rounding, no selection.

See DESIGN.md "Input recipe" for the derivation of every constant.
"""
from .generator import (  # noqa: F401
    Problem, Query, make_config, make_fleet, CONFIG_NAMES, INF, SplitMix64, SharedFleet, make_shared,
    LEVELS, GPU_CLASSES, va_seconds,
)
