"""STORM per-layer attention on the GPU:
tsf_storm_attn(u, ctx, sigma) = u + (1 - g) SelfAttn(u) + g CrossAttn(u, ctx),
g = sigma^2 / (sigma^2 + sigma_data^2) (reading G18), compared with the fp64
oracle (oracle.storm_attention) on the same bf16 inputs within the north-star
gates (max-abs 2e-2, rel-L2 1e-2).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2


def check(got, want, what):
    err = np.abs(got - want).max()
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"{what}: max-abs {err:.3e} rel-L2 {rel:.3e} max|ref| {np.abs(want).max():.2f}")
    assert np.all(np.isfinite(got)) and err <= MAX_ABS and rel <= REL_L2, what


# (B, N, M, H, d): flash self-attention over N, cross-attention over M != N
SHAPES = [(2, 300, 37, 2, 64), (1, 4096, 256, 4, 64), (3, 130, 1, 2, 32), (2, 200, 500, 1, 128),
          (4, 64, 16, 2, 64), (2, 257, 96, 3, 64)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("sigma", [0.0, 0.5, 3.0])
def test_storm_matches_oracle(tsf_lib, shape, sigma):
    B, N, M, H, d = shape
    u = synth.make_x(B, N, H, d, seed=41)
    ctx = synth.make_iid(B, M, H, d, seed=42, role="k")
    layer = tsf_lib.Layer(B, N, H, d)
    y = layer.storm(synth.bits_to_torch(u, "cuda"), synth.bits_to_torch(ctx, "cuda"), sigma, 1.0)
    torch.cuda.synchronize()
    want = oracle.storm_attention(synth.bf16_bits_to_f64(u), synth.bf16_bits_to_f64(ctx), sigma, 1.0)
    check(y.double().cpu().numpy(), want, f"storm sigma={sigma} {shape}")


def test_storm_single_context_token_and_errors(tsf_lib):
    """M = 1: the cross branch returns the context token itself; bad sigma / M rejected."""
    B, N, H, d = 2, 200, 2, 64
    u = synth.make_x(B, N, H, d, seed=43)
    c1 = synth.make_iid(B, 1, H, d, seed=44, role="k")
    layer = tsf_lib.Layer(B, N, H, d)
    uu, cc = synth.bits_to_torch(u, "cuda"), synth.bits_to_torch(c1, "cuda")
    y = layer.storm(uu, cc, 1e6, 1.0).double().cpu().numpy()       # g = 1 - 1e-12
    want = synth.bf16_bits_to_f64(u) + np.broadcast_to(synth.bf16_bits_to_f64(c1), u.shape)
    assert np.abs(y - want).max() <= 2e-5
    for sig, sd in ((-1.0, 1.0), (1.0, 0.0), (float("nan"), 1.0)):
        with pytest.raises(tsf_lib.TsfError) as e:
            layer.storm(uu, cc, sig, sd)
        assert e.value.status == tsf_lib.TSF_ERR_CONFIG
