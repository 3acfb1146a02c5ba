"""The shared seeded input generator (synth/): determinism, shard independence, bf16 RNE."""
import numpy as np
import torch

import synth


def test_bf16_rounding_matches_torch_rne():
    g = np.random.default_rng(5)
    a = np.concatenate([g.normal(0, 3, 100000), [0.0, -0.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -4.0, 65504.0]])
    ours = synth.f64_to_bf16_bits(a)
    ref = torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    back = synth.bf16_bits_to_f64(ours)
    assert np.array_equal(back, torch.from_numpy(ref.view(np.int16)).view(torch.bfloat16).double().numpy())


def test_field_is_deterministic_and_shardable():
    a = synth.make_x(4, 64, 2, 32, seed=1)
    b = synth.make_x(4, 64, 2, 32, seed=1)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, synth.make_x(4, 64, 2, 32, seed=2))
    part = synth.make_x(4, 64, 2, 32, seed=1, frames=[2, 3], tokens=slice(16, 48))
    assert np.array_equal(part, a[2:4, 16:48])


def test_field_statistics_and_clip():
    x = synth.bf16_bits_to_f64(synth.make_x(2, 1024, 4, 64, seed=0))
    assert np.abs(x).max() <= 4.0
    assert 0.7 < x.std() < 1.3
    assert abs(x.mean()) < 0.2


def test_field_advects_one_token_per_frame():
    """Dynamic channels move +1 token in longitude per frame (recipe), so frames differ."""
    x = synth.make_x(3, 256, 1, 32, seed=0)
    assert not np.array_equal(x[0], x[1])


def test_qkv_independent_and_iid_mode():
    q, k, v = synth.make_qkv(2, 64, 2, 32, seed=0)
    assert not np.array_equal(q, k) and not np.array_equal(k, v)
    qi, ki, vi = synth.make_qkv(2, 64, 2, 32, seed=0, kind="iid")
    assert np.array_equal(synth.make_iid(2, 64, 2, 32, seed=0, role="k"), ki)
    qp, _, _ = synth.make_qkv(2, 64, 2, 32, seed=0, peaky=True)
    assert np.abs(synth.bf16_bits_to_f64(qp)).std() > np.abs(synth.bf16_bits_to_f64(q)).std()


def test_grid_shapes_match_configs():
    assert synth.grid_shape(64) == (8, 8)
    assert synth.grid_shape(4096) == (64, 64)
    assert synth.grid_shape(16384) == (128, 128)
    assert synth.grid_shape(1024) == (32, 32)
    assert synth.grid_shape(65536) == (256, 256)
    assert synth.grid_shape(7) == (1, 7)
