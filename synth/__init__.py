"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no bucketing, no planning, no
mapping, no GEMM).  It only draws inputs: routing decisions (top-k expert ids
per token), token activations X and expert weights W.  Both the fp64 oracle
(`oracle/`) and the CUDA path (`paper_2501_16103_b200/`) consume what it
produces; neither imports the other.
"""
from .workloads import (  # noqa: F401
    CONFIGS,
    Config,
    counter_values,
    counter_values_torch,
    make_x,
    make_w,
    make_x_torch,
    make_w_torch,
    route,
    route_balanced,
    route_gumbel,
    route_tiny_a,
    route_paper_best,
    route_paper_worst,
    w_scale_exp,
)
