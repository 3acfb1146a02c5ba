"""Backward pass on the GPU against the fp64 oracle
(oracle.temporal_bwd / spatial_bwd / block_bwd, pinned to torch autograd and
finite differences in tests/test_oracle_pins.py), on the same bf16 inputs.

Tolerance: the gradients carry bf16 roundings of P, dS and the outputs (and,
for the block, of the recomputed X_t): relative L2 error <= 2e-2 per tensor
and max-abs <= 3% of max|ref| (G22).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def check(got, want, what):
    got = got.double().cpu().numpy() if torch.is_tensor(got) else got
    err = np.abs(got - want).max()
    ref = np.abs(want).max()
    if ref == 0.0:   # e.g. K = 1: dq = dk = 0 exactly; the GPU's recomputed P is 1 to rounding
        print(f"{what}: reference is exactly zero, max |got| {err:.3e}")
        assert err <= 1e-5, what
        return
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"{what}: max-abs {err:.3e} ({err / ref:.2%} of max|ref| {ref:.3f}) rel-L2 {rel:.3e}")
    assert np.all(np.isfinite(got)) and rel <= 2e-2 and err <= 3e-2 * ref, what


SHAPES = [(4, 64, 2, 32), (8, 300, 2, 64), (200, 4, 2, 64), (3, 130, 1, 64), (1, 257, 2, 64), (130, 3, 2, 32),
          (5, 260, 2, 128), (150, 4, 1, 128)]   # d = 128 (the C4 head dim): packed and key-tile paths


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("axis", [0, 1], ids=["temporal", "spatial"])
def test_stage_bwd_matches_oracle(tsf_lib, shape, axis):
    K, N, H, d = shape
    qb, kb, vb = synth.make_qkv(K, N, H, d, seed=61, kind="iid")
    dob = synth.make_iid(K, N, H, d, seed=62, role="v")
    layer = tsf_lib.Layer(K, N, H, d)
    dq, dk, dv = layer.attn_bwd(axis, *(synth.bits_to_torch(a, "cuda") for a in (qb, kb, vb, dob)))
    torch.cuda.synchronize()
    fn = oracle.temporal_bwd if axis == 0 else oracle.spatial_bwd
    want = fn(*(synth.bf16_bits_to_f64(a) for a in (qb, kb, vb, dob)))
    for g, w, n in zip((dq, dk, dv), want, ("dq", "dk", "dv")):
        check(g, w, f"{'temporal' if axis == 0 else 'spatial'} bwd {shape} {n}")


@pytest.mark.parametrize("shape", [(4, 64, 2, 32), (8, 300, 2, 64), (6, 260, 2, 64), (200, 4, 2, 64),
                                   (8, 1024, 8, 64)])   # C2-like: K = 8 temporal (packed), N = 1024 spatial
def test_block_bwd_matches_oracle(tsf_lib, shape):
    K, N, H, d = shape
    xb = synth.make_x(K, N, H, d, seed=63)
    dy = np.random.default_rng(64).normal(0.0, 1.0, (K, N, H, d)).astype(np.float32)
    layer = tsf_lib.Layer(K, N, H, d)
    dx = layer.block_bwd(synth.bits_to_torch(xb, "cuda"), torch.from_numpy(dy).cuda())
    torch.cuda.synchronize()
    check(dx, oracle.block_bwd(synth.bf16_bits_to_f64(xb), dy.astype(np.float64)), f"block bwd {shape} dx")


def test_block_bwd_d128(tsf_lib):
    K, N, H, d = 4, 200, 2, 128
    xb = synth.make_x(K, N, H, d, seed=65)
    dy = np.random.default_rng(66).normal(0.0, 1.0, (K, N, H, d)).astype(np.float32)
    layer = tsf_lib.Layer(K, N, H, d)
    dx = layer.block_bwd(synth.bits_to_torch(xb, "cuda"), torch.from_numpy(dy).cuda())
    torch.cuda.synchronize()
    check(dx, oracle.block_bwd(synth.bf16_bits_to_f64(xb), dy.astype(np.float64)), f"block bwd {(K, N, H, d)} dx")


def test_block_bwd_c2_shape(tsf_lib):
    """C2's frame size and context (K = 8, N = 4096, d = 64) at 4 heads, every element."""
    K, N, H, d = 8, 4096, 4, 64
    xb = synth.make_x(K, N, H, d, seed=67)
    dy = np.random.default_rng(68).normal(0.0, 1.0, (K, N, H, d)).astype(np.float32)
    layer = tsf_lib.Layer(K, N, H, d)
    dx = layer.block_bwd(synth.bits_to_torch(xb, "cuda"), torch.from_numpy(dy).cuda())
    torch.cuda.synchronize()
    check(dx, oracle.block_bwd(synth.bf16_bits_to_f64(xb), dy.astype(np.float64)), f"block bwd {(K, N, H, d)} dx")
