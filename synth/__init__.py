"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (tests, bench).

This module holds NO attention arithmetic.  It only draws numbers: a lat-lon
field shaped like the paper's workloads (ERA5-like channels, PAPER.md P:241;
tokens = 2x2 spatial patches of one frame), projected to H*d
features, clipped to +-4 and rounded to bf16 (round-to-nearest-even).  The
recipe is stated in DESIGN.md section "Input recipe".

Both sides receive the same bf16 bit patterns: the CUDA path as a torch
bfloat16 tensor, the oracle as the exact float64 values of those bits.
"""
from .fields import (  # noqa: F401
    Workload,
    CONFIGS,
    grid_shape,
    make_field,
    make_iid,
    make_qkv,
    make_x,
    bf16_bits_to_f64,
    f64_to_bf16_bits,
    bits_to_torch,
    make_block_params,
    block_params_f64,
    BLOCK_PARAM_SHAPES,
)
