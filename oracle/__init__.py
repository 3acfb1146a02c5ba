"""fp64 CPU oracle of TimeSformer's factorized (divided) space-time attention.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or run this
package.  The product path (`paper_2604_16590_b200`) never imports it and it
never imports the product path; the two share no code.  The only shared module
is `synth/` (seeded input generation, no attention arithmetic).

What it computes (section I "Introduction", and Fig. 1 caption
P:38): "temporal attention at each spatial location ... followed by spatial
attention at each time frame", per-layer cost O(K^2 N + K N^2) (P:38, P:74
Table I).  Tokens are one spatial patch of one frame, K frames x N tokens per
frame.  Readings of what the paper leaves open are listed in DESIGN.md
("Readings of the paper"), G1-G17.

Every function is pinned by tests/test_oracle_pins.py (block-mask equivalence
with joint attention, K=1 / N=1 reductions, library SDPA, closed forms,
permutation equivariance, a hand-derived golden example).  No function is
"parity unpinned".
"""
from .attention import (  # noqa: F401
    softmax_rows,
    attend,
    temporal,
    spatial,
    block,
    joint_masked,
    mask_temporal,
    mask_spatial,
    mask_causal_frames,
    joint_rows,
    noise_gate,
    cross,
    storm_attention,
    layer_norm,
    linear,
    gelu,
    full_block,
    attend_bwd,
    temporal_bwd,
    spatial_bwd,
    block_bwd,
    temporal_rows,
    spatial_rows,
    block_rows,
    block_plane,
    flops_tsf,
    flops_spec_convention,
    shard_tokens,
    shard_frames,
    reshard_t2s,
    reshard_s2t,
)
