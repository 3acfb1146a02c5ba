"""Joint (global) attention over all K*N tokens on the GPU:
tsf_joint_attn, unmasked (the ViT global regime, PAPER.md P:52-55 / P:73),
with the temporal and spatial block masks (a GPU-side block-mask check of the
factorization, pin I1 of P:64) and with the causal-frames variant.

Parity: the fp64 oracle (oracle.joint_masked, oracle.joint_rows) on the same
bf16 inputs, max-abs <= 2e-2 and rel-L2 <= 1e-2 (BASELINE.json north_star).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2
MASKS = {0: None, 1: oracle.mask_temporal, 2: oracle.mask_spatial, 3: oracle.mask_causal_frames}


def check(got, want, what):
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - want).max()
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"{what}: max-abs {err:.3e} rel-L2 {rel:.3e} max|ref| {np.abs(want).max():.2f}")
    assert np.all(np.isfinite(got)) and err <= MAX_ABS and rel <= REL_L2, what


@pytest.mark.parametrize("shape", [(4, 64, 2, 32), (3, 100, 2, 64), (2, 200, 1, 128), (5, 20, 2, 64),
                                   (6, 50, 3, 64), (1, 130, 2, 64),
                                   (4, 257, 2, 64), (3, 300, 2, 32)])   # causal: per-frame key prefixes
@pytest.mark.parametrize("mask", [0, 1, 2, 3])
def test_joint_matches_oracle(tsf_lib, shape, mask):
    K, N, H, d = shape
    qb, kb, vb = synth.make_qkv(K, N, H, d, seed=31, kind="iid")
    layer = tsf_lib.Layer(K, N, H, d)
    o = layer.joint(*(synth.bits_to_torch(a, "cuda") for a in (qb, kb, vb)), mask=mask)
    torch.cuda.synchronize()
    m = MASKS[mask](K, N) if MASKS[mask] else None
    want = oracle.joint_masked(*(synth.bf16_bits_to_f64(a) for a in (qb, kb, vb)), m)
    check(o.double().cpu().numpy(), want, f"joint mask={mask} {shape}")


@pytest.mark.parametrize("shape", [(8, 300, 2, 64), (5, 256, 2, 128), (4, 64, 2, 32)])
def test_block_masked_joint_equals_factorized_on_gpu(tsf_lib, shape):
    """Pin I1 on the GPU: joint attention under M_T / M_S equals the temporal /
    spatial kernels (different kernels and tilings: equal within the gate)."""
    K, N, H, d = shape
    q, k, v = (synth.bits_to_torch(a, "cuda") for a in synth.make_qkv(K, N, H, d, seed=32))
    layer = tsf_lib.Layer(K, N, H, d)
    jt = layer.joint(q, k, v, mask=tsf_lib.TSF_MASK_TEMPORAL).double()
    js = layer.joint(q, k, v, mask=tsf_lib.TSF_MASK_SPATIAL).double()
    t = layer.temporal(q, k, v).double()
    s = layer.spatial(q, k, v).double()
    torch.cuda.synchronize()
    for a, b, what in ((jt, t, "temporal"), (js, s, "spatial")):
        err = (a - b).abs().max().item()
        print(f"joint vs factorized {what} {shape}: max |diff| {err:.3e}")
        assert err <= MAX_ABS, what


@pytest.mark.parametrize("causal", [False, True])
def test_joint_c2_size_sampled(tsf_lib, causal):
    """Global attention over all 32768 tokens of C2 (K=8, N=4096, H=16, d=64)."""
    w = synth.CONFIGS["C2"]
    qb, kb, vb = synth.make_qkv(w.K, w.N, w.H, w.d, seed=33)
    layer = tsf_lib.Layer(w.K, w.N, w.H, w.d)
    o = layer.joint(*(synth.bits_to_torch(a, "cuda") for a in (qb, kb, vb)),
                    mask=tsf_lib.TSF_MASK_CAUSAL_FRAMES if causal else tsf_lib.TSF_MASK_NONE)
    torch.cuda.synchronize()
    g = np.random.default_rng(34)
    rows = sorted({(int(g.integers(w.K)), int(g.integers(w.N)), int(g.integers(w.H))) for _ in range(256)})
    ri = torch.tensor(rows)
    got = o[ri[:, 0], ri[:, 1], ri[:, 2]].double().cpu().numpy()
    want = oracle.joint_rows(*(synth.bf16_bits_to_f64(a) for a in (qb, kb, vb)), rows, causal_frames=causal)
    check(got, want, f"joint C2 causal={causal} sampled")


def test_joint_rejects_bad_mask_and_dist(tsf_lib):
    layer = tsf_lib.Layer(2, 64, 1, 64)
    x = torch.zeros((2, 64, 1, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tsf_lib.TsfError) as e:
        layer.joint(x, x, x, mask=7)
    assert e.value.status == tsf_lib.TSF_ERR_CONFIG
    sim = tsf_lib.Layer(2, 64, 1, 64, sim_world=2)
    with pytest.raises(tsf_lib.TsfError) as e:
        sim.joint(x, x, x)
    assert e.value.status == tsf_lib.TSF_ERR_UNSUPPORTED
