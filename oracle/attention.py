"""Plain fp64 numpy implementation of factorized space-time attention.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Arrays are float64 with the
layout [K, N, H, d] (frames, spatial tokens per frame, heads, head dim), row
major, d fastest (BASELINE.json north_star; SPEC.md S:89 row-major order).

Definitions followed, in the paper's order:

* a token is one spatial patch at one frame; K frames x N tokens
* attention over a set of tokens: S = Q K^T s, P = softmax_rows(S), O = P V
  with s = 1/sqrt(d) (reading G4) and softmax exp(S - rowmax)/rowsum
* temporal attention "at each spatial location": one attention per
  (n, h) over the K frames
* spatial attention "at each time frame": one attention per (t, h) over
  the N tokens
* "followed by": temporal first, then spatial.  The block adds each
  stage's output to its input (residual weight 1, reading G5) with identity
  projections (reading G1): X_t = x + T(x,x,x), y = X_t + S(X_t,X_t,X_t)
* global ViT attention over all K*N tokens (Table I row P:73) with a
  block mask, used only to pin the factorized stages (I1)

The only library primitives are numpy's matmul, exp, max and sum.  Groups are
independent, so they are evaluated in batches of independent groups; nothing
inside one group's attention is blocked, fused or reordered.
"""
from __future__ import annotations

import math
from typing import Iterable, Sequence

import numpy as np

_CHUNK_BYTES = 256 << 20   # max bytes of one batch of score matrices


def _check(*arrays: np.ndarray) -> None:
    for a in arrays:
        if a.dtype != np.float64:
            raise TypeError("oracle works in float64")
        if not np.all(np.isfinite(a)):
            raise ValueError("oracle precondition: finite inputs (reading G11)")


def softmax_rows(S: np.ndarray) -> np.ndarray:
    """P[..., i, j] = exp(S_ij - max_j S_ij) / sum_j exp(S_ij - max_j S_ij).

    Rows that are entirely -inf (fully masked) are a precondition violation.
    """
    m = np.max(S, axis=-1, keepdims=True)
    if not np.all(np.isfinite(m)):
        raise ValueError("softmax row with no unmasked entry")
    e = np.exp(S - m)
    return e / np.sum(e, axis=-1, keepdims=True)


def attend(Q: np.ndarray, Kt: np.ndarray, V: np.ndarray, scale: float | None = None,
           return_p: bool = False):
    """Attention of each group on the leading axes: Q, Kt, V are [..., L, d].

    S = Q Kt^T * scale, P = softmax_rows(S), O = P V  (scale = 1/sqrt(d)).
    """
    d = Q.shape[-1]
    s = 1.0 / math.sqrt(d) if scale is None else scale
    S = np.matmul(Q, np.swapaxes(Kt, -1, -2)) * s
    P = softmax_rows(S)
    O = np.matmul(P, V)
    return (O, P) if return_p else O


def _grouped(Qg: np.ndarray, Kg: np.ndarray, Vg: np.ndarray) -> np.ndarray:
    """attend() over groups on axis 0 of [G, L, d] arrays, in batches of groups."""
    G, L, _ = Qg.shape
    per_group = max(1, L * L * 8 * 3)
    step = max(1, _CHUNK_BYTES // per_group)
    out = np.empty_like(Vg)
    for g0 in range(0, G, step):
        out[g0:g0 + step] = attend(Qg[g0:g0 + step], Kg[g0:g0 + step], Vg[g0:g0 + step])
    return out


def temporal(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Temporal attention at each spatial location.

    out[t, n, h, :] = sum_t' softmax_t'( <q[t,n,h], k[t',n,h]> / sqrt(d) ) v[t',n,h, :]
    Groups (n, h); sequence axis t (K frames).  Cost O(K^2 N).
    """
    _check(q, k, v)
    K, N, H, d = q.shape
    to_g = lambda a: a.transpose(1, 2, 0, 3).reshape(N * H, K, d)   # [n,h][t][d]
    o = _grouped(to_g(q), to_g(k), to_g(v))
    return o.reshape(N, H, K, d).transpose(2, 0, 1, 3).copy()


def spatial(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Spatial attention at each time frame.

    out[t, n, h, :] = sum_n' softmax_n'( <q[t,n,h], k[t,n',h]> / sqrt(d) ) v[t,n',h, :]
    Groups (t, h); sequence axis n (N tokens).  Cost O(K N^2).
    """
    _check(q, k, v)
    K, N, H, d = q.shape
    to_g = lambda a: a.transpose(0, 2, 1, 3).reshape(K * H, N, d)   # [t,h][n][d]
    o = _grouped(to_g(q), to_g(k), to_g(v))
    return o.reshape(K, H, N, d).transpose(0, 2, 1, 3).copy()


def block(x: np.ndarray) -> np.ndarray:
    """Divided space-time block: temporal, then spatial ("followed by").

    X_t = x + temporal(x, x, x);  y = X_t + spatial(X_t, X_t, X_t).
    Readings G1 (identity projections), G5 (residual weight 1), G8 (no
    intermediate rounding in the oracle).
    """
    Xt = x + temporal(x, x, x)
    return Xt + spatial(Xt, Xt, Xt)


# ---------------------------------------------------------------------------
# joint attention under a block mask (global ViT) -- pins only
# ---------------------------------------------------------------------------

def mask_temporal(K: int, N: int) -> np.ndarray:
    """M_T[(t,n), (t',n')] = [n == n']: token attends to its own location."""
    n = np.tile(np.arange(N), K)
    return n[:, None] == n[None, :]


def mask_spatial(K: int, N: int) -> np.ndarray:
    """M_S[(t,n), (t',n')] = [t == t']: token attends to its own frame."""
    t = np.repeat(np.arange(K), N)
    return t[:, None] == t[None, :]


def mask_causal_frames(K: int, N: int) -> np.ndarray:
    """M_C[(t,n), (t',n')] = [t' <= t]: every token of frames up to its own.

    Not the paper's regime (temporal context = frames modelled jointly,
    not autoregressive steps); the causal-temporal variant of SURVEY 8(f)
    NEXT-4, a mask over the same global attention.
    """
    t = np.repeat(np.arange(K), N)
    return t[None, :] <= t[:, None]


def joint_masked(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                 mask: np.ndarray | None = None) -> np.ndarray:
    """Attention of every token over all L = K*N tokens, per head.

    Tokens are flattened (t, n) -> t*N + n.  Entries with mask False get -inf
    before the softmax.  mask=None is unmasked global attention.
    """
    _check(q, k, v)
    K, N, H, d = q.shape
    L = K * N
    f = lambda a: a.reshape(L, H, d).transpose(1, 0, 2)          # [h][token][d]
    S = np.matmul(f(q), np.swapaxes(f(k), -1, -2)) / math.sqrt(d)
    if mask is not None:
        S = np.where(mask[None, :, :], S, -np.inf)
    P = softmax_rows(S)
    o = np.matmul(P, f(v))
    return o.transpose(1, 0, 2).reshape(K, N, H, d).copy()


def joint_rows(q, k, v, rows: Iterable[Sequence[int]], causal_frames: bool = False) -> np.ndarray:
    """Rows (t, n, h) of joint_masked(q, k, v, None or mask_causal_frames),
    one by one (any size): row (t, n) attends to all K*N tokens of head h, or
    to the tokens of frames t' <= t.  -> [R, d]"""
    _check(q, k, v)
    K, N, H, d = q.shape
    out = []
    for t, n, h in rows:
        kf = t + 1 if causal_frames else K
        Kt = k[:kf, :, h].reshape(kf * N, d)
        V = v[:kf, :, h].reshape(kf * N, d)
        out.append(attend(q[t, n, h][None], Kt, V)[0])
    return np.array(out)


# ---------------------------------------------------------------------------
# STORM per-layer attention: spatial self-attention on the
# current state plus cross-attention to M compressed history tokens, mixed by
# the noise gate (section IV-B)
# ---------------------------------------------------------------------------

def noise_gate(sigma: float, sigma_data: float) -> float:
    """g(sigma) = sigma^2 / (sigma^2 + sigma_data^2).

    P:379 fixes only the behaviour ("at high noise levels, STORM relies more on
    historical input and temporal cross-attention, while at low noise levels,
    it emphasizes ... spatial self-attention"); the rational form is SPEC.md's
    reading (examples g(0) = 0, g(sigma_data) = 0.5,
    g(3 sigma_data) = 0.9), reading G18.
    """
    if not sigma_data > 0:
        raise ValueError("sigma_data must be > 0")
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    return sigma * sigma / (sigma * sigma + sigma_data * sigma_data)


def cross(q: np.ndarray, kv_k: np.ndarray, kv_v: np.ndarray) -> np.ndarray:
    """Cross-attention of the N query tokens of each (frame, head) over the M
    context tokens of the same (frame, head): q [B, N, H, d], k/v [B, M, H, d]."""
    _check(q, kv_k, kv_v)
    B, N, H, d = q.shape
    M = kv_k.shape[1]
    g = lambda a, L: a.transpose(0, 2, 1, 3).reshape(B * H, L, d)
    o = _grouped_qk(g(q, N), g(kv_k, M), g(kv_v, M))
    return o.reshape(B, H, N, d).transpose(0, 2, 1, 3).copy()


def _grouped_qk(Qg: np.ndarray, Kg: np.ndarray, Vg: np.ndarray) -> np.ndarray:
    """attend() per group with query and key lengths that may differ."""
    G, Lq, d = Qg.shape
    Lk = Kg.shape[1]
    step = max(1, _CHUNK_BYTES // max(1, Lq * Lk * 8 * 3))
    out = np.empty((G, Lq, d))
    for g0 in range(0, G, step):
        out[g0:g0 + step] = attend(Qg[g0:g0 + step], Kg[g0:g0 + step], Vg[g0:g0 + step])
    return out


def storm_attention(u: np.ndarray, ctx: np.ndarray, sigma: float, sigma_data: float) -> np.ndarray:
    """One STORM layer's attention with identity projections (reading G1):

        y = u + (1 - g) SelfAttn_spatial(u) + g CrossAttn(u, ctx),  g = noise_gate(sigma)

    u: [B, N, H, d] current-state tokens (B independent states), ctx:
    [B, M, H, d] compressed temporal representation ("cross-attention
    between the current state and the compressed temporal representation";
    per-layer update form from SPEC.md S:246).
    """
    g = noise_gate(sigma, sigma_data)
    return u + (1.0 - g) * spatial(u, u, u) + g * cross(u, ctx, ctx)


# ---------------------------------------------------------------------------
# sampled rows (any size): an output row depends on its query row and its group
# ---------------------------------------------------------------------------

def temporal_rows(q, k, v, rows: Iterable[Sequence[int]]) -> np.ndarray:
    """Rows (t, n, h) of temporal(q, k, v), computed one by one.  -> [R, d]"""
    out = []
    for t, n, h in rows:
        out.append(attend(q[t, n, h][None], k[:, n, h], v[:, n, h])[0])
    return np.array(out)


def spatial_rows(q, k, v, rows: Iterable[Sequence[int]]) -> np.ndarray:
    """Rows (t, n, h) of spatial(q, k, v), computed one by one.  -> [R, d]"""
    out = []
    for t, n, h in rows:
        out.append(attend(q[t, n, h][None], k[t, :, h], v[t, :, h])[0])
    return np.array(out)


def _xt_plane(x: np.ndarray, t: int, h: int) -> np.ndarray:
    """X_t[t, :, h, :] = x[t, :, h, :] + temporal(x, x, x)[t, :, h, :]  -> [N, d]."""
    xg = x[:, :, h, :].transpose(1, 0, 2)              # [n][t'][d]
    o = attend(xg[:, t:t + 1, :], xg, xg)[:, 0, :]     # query frame t, keys all frames
    return x[t, :, h, :] + o


def block_rows(x: np.ndarray, rows: Iterable[Sequence[int]]) -> np.ndarray:
    """Rows (t, n, h) of block(x).  y[t,n,h] needs X_t[t, :, h, :] (all n)."""
    cache: dict = {}
    out = []
    for t, n, h in rows:
        if (t, h) not in cache:
            cache[(t, h)] = _xt_plane(x, t, h)
        P = cache[(t, h)]
        out.append(P[n] + attend(P[n][None], P, P)[0])
    return np.array(out)


def block_plane(x: np.ndarray, t: int, h: int) -> np.ndarray:
    """The full (t, h) plane y[t, :, h, :] of block(x).  -> [N, d]"""
    P = _xt_plane(x, t, h)
    return P + attend(P, P, P)


# ---------------------------------------------------------------------------
# cost model (P:64 complexity; SPEC.md S:631 convention)
# ---------------------------------------------------------------------------

def flops_spec_convention(K: int, N: int, d: int) -> int:
    """timesformer = 2 K N^2 d + 2 N K^2 d (QK^T only, one head)."""
    return 2 * K * N * N * d + 2 * N * K * K * d


def flops_tsf(K: int, N: int, H: int, d: int) -> int:
    """Reported algorithmic flops: QK^T + PV, multiply-add = 2 (reading G15).

    F = 4 H d (K N^2 + N K^2) = 2 H x flops_spec_convention.
    """
    return 4 * H * d * (K * N * N + N * K * K)


# ---------------------------------------------------------------------------
# distributed semantics (reading G17): pure index permutations, no arithmetic
# ---------------------------------------------------------------------------

def shard_tokens(a: np.ndarray, P: int, p: int) -> np.ndarray:
    """Token shard p of [K, N, H, d]: tokens [p N/P, (p+1) N/P)."""
    N = a.shape[1]
    if N % P:
        raise ValueError("N % P != 0")
    w = N // P
    return a[:, p * w:(p + 1) * w]


def shard_frames(a: np.ndarray, P: int, p: int) -> np.ndarray:
    """Frame shard p of [K, N, H, d]: frames [p K/P, (p+1) K/P)."""
    K = a.shape[0]
    if K % P:
        raise ValueError("K % P != 0")
    w = K // P
    return a[p * w:(p + 1) * w]


def reshard_t2s(token_shards: Sequence[np.ndarray]) -> list:
    """Token-sharded [K, N/P, H, d] x P  ->  frame-sharded [K/P, N, H, d] x P."""
    full = np.concatenate(list(token_shards), axis=1)
    P = len(token_shards)
    return [shard_frames(full, P, p).copy() for p in range(P)]


def reshard_s2t(frame_shards: Sequence[np.ndarray]) -> list:
    """Frame-sharded [K/P, N, H, d] x P  ->  token-sharded [K, N/P, H, d] x P."""
    full = np.concatenate(list(frame_shards), axis=0)
    P = len(frame_shards)
    return [shard_tokens(full, P, p).copy() for p in range(P)]


# ---------------------------------------------------------------------------
# full TimeSformer divided block: per-stage projections,
# pre-LayerNorm, MLP around the factorized attention (reading G21)
# ---------------------------------------------------------------------------

def layer_norm(x: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    """(x - mean) / sqrt(var + eps) * gamma + beta over the last axis (biased variance)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * gamma + beta


def linear(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x W^T + b with W in the [out, in] layout."""
    return np.matmul(x, w.T) + b


def gelu(x: np.ndarray) -> np.ndarray:
    """GELU, exact form 0.5 x (1 + erf(x / sqrt 2))."""
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def full_block(x: np.ndarray, p: dict) -> np.ndarray:
    """TimeSformer divided space-time block (reading G21), x [K, N, H, d]:

        (q, k, v) = split(LN_t(x) Wqkv_t^T + bqkv_t);   X_t = x + T(q, k, v) Wo_t^T + bo_t
        (q, k, v) = split(LN_s(X_t) Wqkv_s^T + bqkv_s); X_s = X_t + S(q, k, v) Wo_s^T + bo_s
        y = X_s + GELU(LN_m(X_s) W1^T + b1) W2^T + b2

    T / S are temporal / spatial attention ("followed by"), split takes
    columns [0, D), [D, 2D), [2D, 3D) as q, k, v with D = H d and head h at
    columns [h d, (h+1) d) of each.  p holds float64 arrays keyed as in
    synth.make_block_params.
    """
    _check(x)
    K, N, H, d = x.shape
    D = H * d
    xs = x.reshape(K, N, D)

    def qkv(h, w, b):
        t = linear(h, w, b)
        return tuple(t[..., i * D:(i + 1) * D].reshape(K, N, H, d) for i in range(3))

    q, k, v = qkv(layer_norm(xs, p["ln_t_g"], p["ln_t_b"]), p["w_qkv_t"], p["b_qkv_t"])
    xt = xs + linear(temporal(q, k, v).reshape(K, N, D), p["w_o_t"], p["b_o_t"])
    q, k, v = qkv(layer_norm(xt, p["ln_s_g"], p["ln_s_b"]), p["w_qkv_s"], p["b_qkv_s"])
    xsp = xt + linear(spatial(q, k, v).reshape(K, N, D), p["w_o_s"], p["b_o_s"])
    m = gelu(linear(layer_norm(xsp, p["ln_m_g"], p["ln_m_b"]), p["w_1"], p["b_1"]))
    y = xsp + linear(m, p["w_2"], p["b_2"])
    return y.reshape(K, N, H, d)


# ---------------------------------------------------------------------------
# backward pass: gradients of the attention stages and of
# the block, from the definitions (P:64 forward; training)
# ---------------------------------------------------------------------------

def attend_bwd(Q: np.ndarray, Kt: np.ndarray, V: np.ndarray, dO: np.ndarray):
    """Gradients of O = softmax(Q Kt^T / sqrt d) V for groups on the leading axes:

        P = softmax_rows(S), dV = P^T dO, dP = dO V^T,
        dS = P * (dP - rowsum(dP * P)),  dQ = dS Kt / sqrt d,  dK = dS^T Q / sqrt d.
    """
    d = Q.shape[-1]
    s = 1.0 / math.sqrt(d)
    S = np.matmul(Q, np.swapaxes(Kt, -1, -2)) * s
    P = softmax_rows(S)
    dV = np.matmul(np.swapaxes(P, -1, -2), dO)
    dP = np.matmul(dO, np.swapaxes(V, -1, -2))
    dS = P * (dP - np.sum(dP * P, axis=-1, keepdims=True))
    dQ = np.matmul(dS, Kt) * s
    dK = np.matmul(np.swapaxes(dS, -1, -2), Q) * s
    return dQ, dK, dV


def _stage_bwd(q, k, v, do, axis):
    """Gradients of the temporal (axis 0) or spatial (axis 1) stage, [K, N, H, d]."""
    _check(q, k, v, do)
    K, N, H, d = q.shape
    if axis == 0:
        g = lambda a: a.transpose(1, 2, 0, 3).reshape(N * H, K, d)
        ug = lambda a: a.reshape(N, H, K, d).transpose(2, 0, 1, 3)
    else:
        g = lambda a: a.transpose(0, 2, 1, 3).reshape(K * H, N, d)
        ug = lambda a: a.reshape(K, H, N, d).transpose(0, 2, 1, 3)
    dq, dk, dv = attend_bwd(g(q), g(k), g(v), g(do))
    return ug(dq).copy(), ug(dk).copy(), ug(dv).copy()


def temporal_bwd(q, k, v, do):
    """(dq, dk, dv) of temporal(q, k, v) for the output gradient do."""
    return _stage_bwd(q, k, v, do, 0)


def spatial_bwd(q, k, v, do):
    """(dq, dk, dv) of spatial(q, k, v) for the output gradient do."""
    return _stage_bwd(q, k, v, do, 1)


def block_bwd(x: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """dx of block(x) = X_t + S(X_t, X_t, X_t), X_t = x + T(x, x, x), for dy:

        dX_t = dy + (dq + dk + dv of S at X_t),  dx = dX_t + (dq + dk + dv of T at x)
    (q = k = v = the stage input, so its gradient is the sum of the three).
    """
    _check(x, dy)
    xt = x + temporal(x, x, x)
    a, b, c = spatial_bwd(xt, xt, xt, dy)
    dxt = dy + a + b + c
    a, b, c = temporal_bwd(x, x, x, dxt)
    return dxt + a + b + c
