"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the pin from SURVEY.md 8(c) / DESIGN.md "Oracle pins" it
implements.  A plausible mistake in oracle/ (a transposed axis, a missing
scale, a wrong residual, a softmax over the wrong axis) fails at least one.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")
RNG = np.random.default_rng(20260418)


def rand(*shape, scale=1.0):
    return RNG.normal(0.0, scale, shape)


SHAPES = [(3, 4, 2, 4), (1, 5, 1, 3), (4, 1, 2, 2), (2, 3, 1, 8), (5, 6, 3, 2)]


# --- I1: block-mask equivalence with joint attention over all K*N tokens ----

@pytest.mark.parametrize("shape", SHAPES)
def test_I1_temporal_equals_joint_under_temporal_mask(shape):
    q, k, v = rand(*shape), rand(*shape), rand(*shape)
    K, N = shape[:2]
    ref = oracle.joint_masked(q, k, v, oracle.mask_temporal(K, N))
    np.testing.assert_allclose(oracle.temporal(q, k, v), ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape", SHAPES)
def test_I1_spatial_equals_joint_under_spatial_mask(shape):
    q, k, v = rand(*shape), rand(*shape), rand(*shape)
    K, N = shape[:2]
    ref = oracle.joint_masked(q, k, v, oracle.mask_spatial(K, N))
    np.testing.assert_allclose(oracle.spatial(q, k, v), ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape", SHAPES)
def test_I1_block_equals_masked_joint_composition(shape):
    x = rand(*shape)
    K, N = shape[:2]
    xt = x + oracle.joint_masked(x, x, x, oracle.mask_temporal(K, N))
    ref = xt + oracle.joint_masked(xt, xt, xt, oracle.mask_spatial(K, N))
    np.testing.assert_allclose(oracle.block(x), ref, rtol=0, atol=1e-12)


def test_joint_unmasked_matches_brute_force_loops():
    """Tiny brute force with math.exp loops (independent of numpy's matmul)."""
    K, N, H, d = 2, 2, 1, 3
    q, k, v = rand(K, N, H, d), rand(K, N, H, d), rand(K, N, H, d)
    toks = [(t, n) for t in range(K) for n in range(N)]
    out = np.zeros_like(q)
    for h in range(H):
        for (t, n) in toks:
            w = [math.exp(sum(q[t, n, h, i] * k[a, b, h, i] for i in range(d)) / math.sqrt(d))
                 for (a, b) in toks]
            z = sum(w)
            for i in range(d):
                out[t, n, h, i] = sum(wj * v[a, b, h, i] for wj, (a, b) in zip(w, toks)) / z
    np.testing.assert_allclose(oracle.joint_masked(q, k, v), out, rtol=0, atol=1e-12)


def test_joint_causal_frames_matches_brute_force_loops():
    """Causal-in-time joint attention (SURVEY NEXT-4 variant): token (t, n) attends
    to every (t', n') with t' <= t; tiny brute force with math.exp loops."""
    K, N, H, d = 3, 2, 2, 3
    q, k, v = rand(K, N, H, d), rand(K, N, H, d), rand(K, N, H, d)
    out = np.zeros_like(q)
    for h in range(H):
        for t in range(K):
            for n in range(N):
                keys = [(a, b) for a in range(t + 1) for b in range(N)]
                w = [math.exp(sum(q[t, n, h, i] * k[a, b, h, i] for i in range(d)) / math.sqrt(d)) for a, b in keys]
                z = sum(w)
                for i in range(d):
                    out[t, n, h, i] = sum(wj * v[a, b, h, i] for wj, (a, b) in zip(w, keys)) / z
    np.testing.assert_allclose(oracle.joint_masked(q, k, v, oracle.mask_causal_frames(K, N)), out,
                               rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape", [(3, 5, 2, 4), (1, 7, 1, 8), (4, 1, 2, 2)])
def test_joint_causal_frames_special_cases(shape):
    """Frame 0 attends only to itself (= spatial attention of frame 0); the last
    frame attends to everything (= unmasked joint attention); K = 1 is spatial."""
    q, k, v = rand(*shape), rand(*shape), rand(*shape)
    K, N = shape[:2]
    c = oracle.joint_masked(q, k, v, oracle.mask_causal_frames(K, N))
    np.testing.assert_allclose(c[0], oracle.spatial(q, k, v)[0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(c[K - 1], oracle.joint_masked(q, k, v)[K - 1], rtol=0, atol=1e-12)
    m = oracle.mask_causal_frames(K, N)
    assert m.sum() == N * N * K * (K + 1) // 2                 # lower block triangle incl. diagonal


@pytest.mark.parametrize("causal", [False, True])
def test_joint_rows_match_full_joint(causal):
    K, N, H, d = 3, 4, 2, 4
    q, k, v = rand(K, N, H, d), rand(K, N, H, d), rand(K, N, H, d)
    full = oracle.joint_masked(q, k, v, oracle.mask_causal_frames(K, N) if causal else None)
    rows = [(0, 0, 0), (2, 3, 1), (1, 2, 0), (2, 0, 1)]
    got = oracle.joint_rows(q, k, v, rows, causal_frames=causal)
    np.testing.assert_allclose(got, np.array([full[t, n, h] for t, n, h in rows]), rtol=0, atol=1e-12)


# --- library routine: torch SDPA in fp64 on CPU -----------------------------

def sdpa(q, k, v):
    """[G, L, d] fp64 through torch.nn.functional.scaled_dot_product_attention."""
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))[None]
    return torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v))[0].numpy()


@pytest.mark.parametrize("causal", [False, True])
def test_joint_matches_library_sdpa(causal):
    """Unmasked global attention over all K*N tokens and its
    causal-frame variant = torch SDPA fp64 (boolean attn_mask)."""
    K, N, H, d = 3, 5, 2, 8
    q, k, v = rand(K, N, H, d), rand(K, N, H, d), rand(K, N, H, d)
    g = lambda a: torch.from_numpy(np.ascontiguousarray(a.reshape(K * N, H, d).transpose(1, 0, 2)))
    m = torch.from_numpy(oracle.mask_causal_frames(K, N)) if causal else None
    ref = torch.nn.functional.scaled_dot_product_attention(g(q), g(k), g(v), attn_mask=m).numpy()
    ref = ref.transpose(1, 0, 2).reshape(K, N, H, d)
    got = oracle.joint_masked(q, k, v, oracle.mask_causal_frames(K, N) if causal else None)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape", [(6, 7, 3, 16), (1, 33, 2, 32), (9, 1, 2, 64)])
def test_temporal_matches_library_sdpa(shape):
    q, k, v = rand(*shape), rand(*shape), rand(*shape)
    K, N, H, d = shape
    g = lambda a: a.transpose(1, 2, 0, 3).reshape(N * H, K, d)
    ref = sdpa(g(q), g(k), g(v)).reshape(N, H, K, d).transpose(2, 0, 1, 3)
    np.testing.assert_allclose(oracle.temporal(q, k, v), ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape", [(6, 7, 3, 16), (2, 65, 2, 32), (1, 40, 1, 64)])
def test_spatial_matches_library_sdpa(shape):
    q, k, v = rand(*shape), rand(*shape), rand(*shape)
    K, N, H, d = shape
    g = lambda a: a.transpose(0, 2, 1, 3).reshape(K * H, N, d)
    ref = sdpa(g(q), g(k), g(v)).reshape(K, H, N, d).transpose(0, 2, 1, 3)
    np.testing.assert_allclose(oracle.spatial(q, k, v), ref, rtol=0, atol=1e-12)


# --- I2 / I3: degenerate sizes ---------------------------------------------

def test_I2_K1_temporal_is_identity_on_v_exactly():
    q, k, v = rand(1, 9, 2, 8), rand(1, 9, 2, 8), rand(1, 9, 2, 8)
    assert np.array_equal(oracle.temporal(q, k, v), v)


def test_I3_N1_spatial_is_identity_on_v_exactly():
    q, k, v = rand(7, 1, 2, 8), rand(7, 1, 2, 8), rand(7, 1, 2, 8)
    assert np.array_equal(oracle.spatial(q, k, v), v)


def test_I2_K1_block_closed_form():
    """K=1: X_t = x + x = 2x, y = 2x + SDPA(2x) per head (library routine)."""
    x = rand(1, 11, 2, 8)
    xt = 2 * x
    g = xt[0].transpose(1, 0, 2)                      # [h][n][d]
    ref = xt + sdpa(g, g, g).transpose(1, 0, 2)[None]
    np.testing.assert_allclose(oracle.block(x), ref, rtol=0, atol=1e-12)


# --- I4: permutation equivariance ------------------------------------------

@pytest.mark.parametrize("fn", ["temporal", "spatial"])
def test_I4_permutation_equivariance(fn):
    f = getattr(oracle, fn)
    q, k, v = rand(5, 6, 2, 4), rand(5, 6, 2, 4), rand(5, 6, 2, 4)
    pn, pk = RNG.permutation(6), RNG.permutation(5)
    base = f(q, k, v)
    np.testing.assert_allclose(f(q[:, pn], k[:, pn], v[:, pn]), base[:, pn], atol=1e-12, rtol=0)
    np.testing.assert_allclose(f(q[pk], k[pk], v[pk]), base[pk], atol=1e-12, rtol=0)


def test_I4_block_permutation_equivariance():
    x = rand(4, 6, 2, 4)
    pn, pk = RNG.permutation(6), RNG.permutation(4)
    base = oracle.block(x)
    np.testing.assert_allclose(oracle.block(x[:, pn]), base[:, pn], atol=1e-12, rtol=0)
    np.testing.assert_allclose(oracle.block(x[pk]), base[pk], atol=1e-12, rtol=0)


def test_I4_heads_are_independent():
    x = rand(3, 5, 3, 4)
    y = oracle.block(x)
    for h in range(3):
        np.testing.assert_allclose(oracle.block(x[:, :, h:h + 1]), y[:, :, h:h + 1], atol=1e-12, rtol=0)


# --- I5: softmax rows sum to one -------------------------------------------

def test_I5_rows_sum_to_one():
    q, k, v = rand(4, 37, 8, scale=3.0), rand(4, 37, 8, scale=3.0), rand(4, 37, 8)
    _, P = oracle.attend(q, k, v, return_p=True)
    assert np.max(np.abs(P.sum(-1) - 1.0)) <= 1e-13
    assert np.all(P >= 0)


# --- I6: closed forms -------------------------------------------------------

def test_I6_zero_query_gives_mean_of_v():
    k, v = rand(4, 5, 2, 8), rand(4, 5, 2, 8)
    q = np.zeros_like(k)
    np.testing.assert_allclose(oracle.temporal(q, k, v), np.broadcast_to(v.mean(0, keepdims=True), v.shape), atol=1e-12, rtol=0)
    np.testing.assert_allclose(oracle.spatial(q, k, v), np.broadcast_to(v.mean(1, keepdims=True), v.shape), atol=1e-12, rtol=0)


def test_I6_equal_keys_give_mean_of_v():
    q, v = rand(4, 5, 2, 8), rand(4, 5, 2, 8)
    kt = np.broadcast_to(rand(1, 5, 2, 8), q.shape).copy()      # same key on every frame
    np.testing.assert_allclose(oracle.temporal(q, kt, v), np.broadcast_to(v.mean(0, keepdims=True), v.shape), atol=1e-12, rtol=0)


def test_I6_identical_frames_temporal_returns_frame():
    """All frames identical -> softmax uniform over equal keys -> x[0]."""
    f = rand(1, 6, 2, 8)
    x = np.repeat(f, 5, axis=0)
    np.testing.assert_allclose(oracle.temporal(x, x, x), x, atol=1e-12, rtol=0)


def test_I6_key_shift_invariance():
    q, k, v = rand(4, 5, 2, 8), rand(4, 5, 2, 8), rand(4, 5, 2, 8)
    # temporal: a shift constant along the frame axis adds a per-row constant to S
    c_t = rand(1, 5, 2, 8)
    np.testing.assert_allclose(oracle.temporal(q, k + c_t, v), oracle.temporal(q, k, v), atol=1e-11, rtol=0)
    c_s = rand(4, 1, 2, 8)
    np.testing.assert_allclose(oracle.spatial(q, k + c_s, v), oracle.spatial(q, k, v), atol=1e-11, rtol=0)


def test_I6_linear_in_v_and_convex():
    q, k, v1, v2 = (rand(4, 6, 2, 8) for _ in range(4))
    for f in (oracle.temporal, oracle.spatial):
        np.testing.assert_allclose(f(q, k, 2.0 * v1 - 3.0 * v2), 2.0 * f(q, k, v1) - 3.0 * f(q, k, v2), atol=1e-11, rtol=0)
    o = oracle.temporal(q, k, v1)
    assert np.all(o <= v1.max(0, keepdims=True) + 1e-12) and np.all(o >= v1.min(0, keepdims=True) - 1e-12)
    o = oracle.spatial(q, k, v1)
    assert np.all(o <= v1.max(1, keepdims=True) + 1e-12) and np.all(o >= v1.min(1, keepdims=True) - 1e-12)


# --- I7: large-logit limit ---------------------------------------------------

def test_I7_large_logit_selects_argmax():
    K, N, H, d = 1, 7, 1, 4
    g = np.random.default_rng(7)                          # own stream: independent of test order
    k = g.normal(size=(K, N, H, d))
    k /= np.linalg.norm(k, axis=-1, keepdims=True)        # unit keys: q = 1e3 k_3 has a unique argmax n = 3
    v = g.normal(size=(K, N, H, d))
    q = np.broadcast_to(k[:, 3:4], k.shape) * 1e3
    o = oracle.spatial(q, k, v)
    np.testing.assert_allclose(o, np.broadcast_to(v[:, 3:4], v.shape), atol=1e-9, rtol=0)


# --- golden, hand-derived (tests/golden/hand_examples.json) ------------------

def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_golden_temporal_k2():
    g = golden()["temporal_k2"]
    o = oracle.temporal(*(np.array(g[n], dtype=np.float64) for n in "qkv"))
    np.testing.assert_allclose(o, np.array(g["out"]), atol=1e-15, rtol=0)


def test_golden_spatial_n3():
    g = golden()["spatial_n3"]
    o = oracle.spatial(*(np.array(g[n], dtype=np.float64) for n in "qkv"))
    np.testing.assert_allclose(o, np.array(g["out"]), atol=g["tol"], rtol=0)


def test_golden_block_k2_n1():
    g = golden()["block_k2_n1"]
    y = oracle.block(np.array(g["x"], dtype=np.float64))
    np.testing.assert_allclose(y, np.array(g["y"]), atol=g["tol"], rtol=0)


def test_I8_flop_model_spec_example():
    g = golden()["flops_spec_example"]
    assert oracle.flops_spec_convention(g["K"], g["N"], g["d"]) == g["spec_flops"]
    assert oracle.flops_tsf(g["K"], g["N"], 1, g["d"]) == g["tsf_flops_H1"]


def test_I8_flop_model_counts_matmul_macs():
    """Count the multiply-adds the oracle's matmuls perform, by shape."""
    K, N, H, d = 3, 5, 2, 4
    macs = H * (N * (K * K * d + K * K * d) + K * (N * N * d + N * N * d))
    assert oracle.flops_tsf(K, N, H, d) == 2 * macs


# --- sampled-row evaluation equals the full oracle -------------------------

def test_sampled_rows_match_full():
    K, N, H, d = 4, 9, 3, 8
    q, k, v, x = (rand(K, N, H, d) for _ in range(4))
    rows = [(0, 0, 0), (3, 8, 2), (1, 4, 1), (2, 7, 0)]
    T, S, B = oracle.temporal(q, k, v), oracle.spatial(q, k, v), oracle.block(x)
    pick = lambda a: np.array([a[t, n, h] for t, n, h in rows])
    np.testing.assert_allclose(oracle.temporal_rows(q, k, v, rows), pick(T), atol=1e-12, rtol=0)
    np.testing.assert_allclose(oracle.spatial_rows(q, k, v, rows), pick(S), atol=1e-12, rtol=0)
    np.testing.assert_allclose(oracle.block_rows(x, rows), pick(B), atol=1e-12, rtol=0)
    np.testing.assert_allclose(oracle.block_plane(x, 2, 1), B[2, :, 1], atol=1e-12, rtol=0)


# --- distributed semantics: reshard is a pure permutation ------------------

@pytest.mark.parametrize("P", [1, 2, 4])
def test_reshard_is_index_permutation(P):
    a = rand(8, 12, 2, 4)
    tok = [oracle.shard_tokens(a, P, p) for p in range(P)]
    fr = oracle.reshard_t2s(tok)
    for p in range(P):
        assert np.array_equal(fr[p], a[p * 8 // P:(p + 1) * 8 // P])
    back = oracle.reshard_s2t(fr)
    for p in range(P):
        assert np.array_equal(back[p], tok[p])


def test_sharded_block_equals_block():
    """O5: temporal on token shards, reshard, spatial on frame shards == block."""
    x = rand(4, 6, 2, 4)
    P = 2
    xt = [s + oracle.temporal(s, s, s) for s in (oracle.shard_tokens(x, P, p) for p in range(P))]
    fr = oracle.reshard_t2s(xt)
    y = np.concatenate([f + oracle.spatial(f, f, f) for f in fr], axis=0)
    np.testing.assert_allclose(y, oracle.block(x), atol=1e-12, rtol=0)


def test_oracle_rejects_non_finite():
    q = rand(2, 3, 1, 4)
    q[0, 0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        oracle.temporal(q, q, q)


# --- STORM per-layer attention (NEXT-3) ------------------------------------

def test_noise_gate_spec_examples():
    """SPEC.md S:233-235 printed values; monotone, g(0) = 0, g -> 1."""
    assert oracle.noise_gate(0.0, 0.7) == 0.0
    assert oracle.noise_gate(0.7, 0.7) == 0.5
    assert abs(oracle.noise_gate(2.1, 0.7) - 0.9) < 1e-15
    gs = [oracle.noise_gate(s, 1.0) for s in np.linspace(0, 50, 101)]
    assert all(b > a for a, b in zip(gs, gs[1:])) and gs[-1] > 0.999
    with pytest.raises(ValueError):
        oracle.noise_gate(1.0, 0.0)


def test_cross_matches_library_sdpa():
    """Cross-attention with query and key lengths that differ = torch SDPA fp64."""
    B, N, M, H, d = 2, 7, 5, 3, 8
    q, k, v = rand(B, N, H, d), rand(B, M, H, d), rand(B, M, H, d)
    g = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 1, 3)))
    ref = torch.nn.functional.scaled_dot_product_attention(g(q), g(k), g(v)).numpy().transpose(0, 2, 1, 3)
    np.testing.assert_allclose(oracle.cross(q, k, v), ref, rtol=0, atol=1e-12)


def test_storm_special_cases():
    B, N, M, H, d = 2, 6, 4, 2, 8
    u, ctx = rand(B, N, H, d), rand(B, M, H, d)
    # sigma = 0: pure spatial self-attention on the current state (the block's spatial stage)
    np.testing.assert_allclose(oracle.storm_attention(u, ctx, 0.0, 1.0), u + oracle.spatial(u, u, u),
                               rtol=0, atol=1e-12)
    # one context token: cross-attention returns it exactly (single key, weight 1)
    c1 = rand(B, 1, H, d)
    g = oracle.noise_gate(2.0, 1.0)
    want = u + (1 - g) * oracle.spatial(u, u, u) + g * np.broadcast_to(c1, u.shape)
    np.testing.assert_allclose(oracle.storm_attention(u, c1, 2.0, 1.0), want, rtol=0, atol=1e-12)
    # context = the state itself: cross = self, y = u + spatial(u) for every sigma
    np.testing.assert_allclose(oracle.storm_attention(u, u, 3.0, 1.0), u + oracle.spatial(u, u, u),
                               rtol=0, atol=1e-12)
    # permuting the context tokens changes nothing (keys are a set)
    perm = np.random.default_rng(3).permutation(M)
    np.testing.assert_allclose(oracle.storm_attention(u, ctx[:, perm], 1.5, 1.0),
                               oracle.storm_attention(u, ctx, 1.5, 1.0), rtol=0, atol=1e-12)


# --- full divided block (NEXT-1, reading G21) -------------------------------

def _torch_full_block(x, p):
    """The same block composed from torch library modules in fp64 (layer_norm,
    linear, SDPA per group, exact GELU): an implementation independent of the
    oracle's numpy arithmetic."""
    import torch.nn.functional as F
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    K, N, H, d = x.shape
    D = H * d
    P = {k: t(v) for k, v in p.items()}
    X = t(x).reshape(K, N, D)

    def proj(h, w, b):
        z = F.linear(h, w, b)
        return [z[..., i * D:(i + 1) * D].reshape(K, N, H, d) for i in range(3)]

    def attn(q, k, v, axis):      # axis 0: over frames (temporal), 1: over tokens (spatial)
        perm = (1, 2, 0, 3) if axis == 0 else (0, 2, 1, 3)
        inv = (2, 0, 1, 3) if axis == 0 else (0, 2, 1, 3)
        o = F.scaled_dot_product_attention(q.permute(*perm), k.permute(*perm), v.permute(*perm))
        return o.permute(*inv).reshape(K, N, D)

    q, k, v = proj(F.layer_norm(X, (D,), P["ln_t_g"], P["ln_t_b"], 1e-5), P["w_qkv_t"], P["b_qkv_t"])
    Xt = X + F.linear(attn(q, k, v, 0), P["w_o_t"], P["b_o_t"])
    q, k, v = proj(F.layer_norm(Xt, (D,), P["ln_s_g"], P["ln_s_b"], 1e-5), P["w_qkv_s"], P["b_qkv_s"])
    Xs = Xt + F.linear(attn(q, k, v, 1), P["w_o_s"], P["b_o_s"])
    m = F.gelu(F.linear(F.layer_norm(Xs, (D,), P["ln_m_g"], P["ln_m_b"], 1e-5), P["w_1"], P["b_1"]))
    return (Xs + F.linear(m, P["w_2"], P["b_2"])).reshape(K, N, H, d).numpy()


def _params(H, d, F, seed=7):
    import synth
    return synth.block_params_f64(synth.make_block_params(H, d, F, seed))


@pytest.mark.parametrize("shape", [(3, 5, 2, 4), (1, 6, 1, 8), (4, 1, 2, 4)])
def test_full_block_matches_torch_library_composition(shape):
    K, N, H, d = shape
    x = rand(*shape)
    p = _params(H, d, 4 * H * d)
    np.testing.assert_allclose(oracle.full_block(x, p), _torch_full_block(x, p), rtol=0, atol=1e-11)


def test_full_block_zero_output_projections_is_identity():
    """W_o, b_o of both stages and W_2, b_2 zero: every branch adds exactly zero."""
    K, N, H, d = 3, 4, 2, 4
    p = _params(H, d, 32)
    for k in ("w_o_t", "b_o_t", "w_o_s", "b_o_s", "w_2", "b_2"):
        p[k] = np.zeros_like(p[k])
    x = rand(K, N, H, d)
    np.testing.assert_array_equal(oracle.full_block(x, p), x)


def test_full_block_permutation_equivariance():
    K, N, H, d = 3, 5, 2, 4
    p = _params(H, d, 32)
    x = rand(K, N, H, d)
    y = oracle.full_block(x, p)
    pn, pk = np.random.default_rng(5).permutation(N), np.random.default_rng(6).permutation(K)
    np.testing.assert_allclose(oracle.full_block(x[:, pn], p), y[:, pn], rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.full_block(x[pk], p), y[pk], rtol=0, atol=1e-12)


def test_layer_norm_and_gelu_closed_forms():
    x = np.array([[1.0, 2.0, 3.0, 6.0]])
    # mean 3, biased variance 3.5
    want = (x - 3.0) / math.sqrt(3.5 + 1e-5)
    np.testing.assert_allclose(oracle.layer_norm(x, np.ones(4), np.zeros(4)), want, rtol=0, atol=1e-15)
    assert oracle.gelu(np.array([0.0]))[0] == 0.0
    # GELU(1) = 0.5 (1 + erf(1/sqrt 2)) = Phi(1) = 0.8413447460685429 (standard normal CDF)
    assert abs(oracle.gelu(np.array([1.0]))[0] - 0.8413447460685429) < 1e-15


# --- backward (NEXT-2) -------------------------------------------------------

def _autograd_stage(q, k, v, do, axis):
    """torch autograd through SDPA in fp64 (library routine)."""
    K, N, H, d = q.shape
    perm = (1, 2, 0, 3) if axis == 0 else (0, 2, 1, 3)
    inv = (2, 0, 1, 3) if axis == 0 else (0, 2, 1, 3)
    ts = [torch.from_numpy(np.ascontiguousarray(a)).requires_grad_(True) for a in (q, k, v)]
    o = torch.nn.functional.scaled_dot_product_attention(*(t.permute(*perm) for t in ts)).permute(*inv)
    o.backward(torch.from_numpy(do))
    return [t.grad.numpy() for t in ts]


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("shape", [(5, 6, 2, 4), (1, 7, 1, 8), (3, 1, 2, 4)])
def test_stage_bwd_matches_library_autograd(axis, shape):
    q, k, v, do = (rand(*shape) for _ in range(4))
    got = (oracle.temporal_bwd if axis == 0 else oracle.spatial_bwd)(q, k, v, do)
    for g, w in zip(got, _autograd_stage(q, k, v, do, axis)):
        np.testing.assert_allclose(g, w, rtol=0, atol=1e-11)


def test_block_bwd_matches_finite_differences():
    """Central differences of <dy, block(x)> in fp64 (independent of any autograd)."""
    K, N, H, d = 3, 4, 1, 3
    x, dy = rand(K, N, H, d), rand(K, N, H, d)
    dx = oracle.block_bwd(x, dy)
    f = lambda a: float(np.sum(dy * oracle.block(a)))
    h = 1e-6
    num = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        e = np.zeros_like(x)
        e[idx] = h
        num[idx] = (f(x + e) - f(x - e)) / (2 * h)
    np.testing.assert_allclose(dx, num, rtol=0, atol=1e-7)


def test_block_bwd_matches_library_autograd():
    K, N, H, d = 4, 5, 2, 4
    x, dy = rand(K, N, H, d), rand(K, N, H, d)
    xt_ = torch.from_numpy(x).requires_grad_(True)
    sdpa = torch.nn.functional.scaled_dot_product_attention
    t = lambda a: sdpa(a.permute(1, 2, 0, 3), a.permute(1, 2, 0, 3), a.permute(1, 2, 0, 3)).permute(2, 0, 1, 3)
    s_ = lambda a: sdpa(a.permute(0, 2, 1, 3), a.permute(0, 2, 1, 3), a.permute(0, 2, 1, 3)).permute(0, 2, 1, 3)
    Xt = xt_ + t(xt_)
    y = Xt + s_(Xt)
    y.backward(torch.from_numpy(dy))
    np.testing.assert_allclose(oracle.block_bwd(x, dy), xt_.grad.numpy(), rtol=0, atol=1e-11)


def test_stage_bwd_closed_forms():
    """K = 1: temporal output = v, so dv = do and dq = dk = 0 exactly (one key, weight 1)."""
    q, k, v, do = (rand(1, 5, 2, 4) for _ in range(4))
    dq, dk, dv = oracle.temporal_bwd(q, k, v, do)
    np.testing.assert_array_equal(dv, do)
    assert np.all(dq == 0) and np.all(dk == 0)
