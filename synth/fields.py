"""Synthetic lat-lon fields x temporal context, rounded to bf16.

Recipe:

* Token grid n_lat x n_lon (lat-major, row-major), each token
  a p x p = 2 x 2 patch of a (2 n_lat) x (2 n_lon) pixel grid (PAPER.md P:52,
  2x2 patches P:509).
* C = 6 channels per pixel, like ERA5's six variables: three static
  ones (orography-like random field, land-sea-like threshold of a second field,
  sin(latitude)) and three dynamic ones.  A dynamic channel is a sum of M = 32
  random Fourier modes with a squared-exponential spectrum (correlation length
  about 4 tokens), advected by +1 token in longitude per frame (periodic), plus
  N(0, 0.1^2) pixel noise.
* The p*p*C = 24 patch features go through a fixed seeded Gaussian projection
  to H*d features (one projection per role: x, q, k, v), are clipped to +-4 and
  rounded to bf16 with round-to-nearest-even.

Every random stream is keyed by (seed, role, frame) so any frame range or token
range can be generated alone and equals the same slice of the full tensor: a
rank can build its shard without building the whole field.

No attention arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

N_MODES = 32          # Fourier modes per dynamic channel
CORR_TOKENS = 4.0     # correlation length, tokens
PATCH = 2             # p: pixels per token side ("2x2")
N_CHANNELS = 6        # ERA5-like channel count
NOISE_STD = 0.1
CLIP = 4.0
PROJ_SEED = 1234
ROLES = {"x": 0, "q": 1, "k": 2, "v": 3}


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    K: int
    N: int
    H: int
    d: int

    @property
    def E(self) -> int:
        return self.K * self.N * self.H * self.d


# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": Workload("C1", 4, 64, 2, 32),
    "C2": Workload("C2", 8, 4096, 16, 64),
    "C3": Workload("C3", 32, 16384, 16, 64),
    "C4": Workload("C4", 128, 65536, 16, 128),
    "C5": Workload("C5", 1024, 1024, 8, 64),
}


def grid_shape(N: int) -> tuple[int, int]:
    """n_lat x n_lon = N with n_lat the largest divisor of N not above sqrt(N)."""
    n_lat = 1
    for a in range(1, int(math.isqrt(N)) + 1):
        if N % a == 0:
            n_lat = a
    return n_lat, N // n_lat


# ---------------------------------------------------------------------------
# bf16 bit handling (round-to-nearest-even), numpy only
# ---------------------------------------------------------------------------

def f64_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round to float32 (RNE), then to bf16 (RNE); returns the uint16 bit patterns.

    Inputs must be finite.  Double rounding f64 -> f32 -> bf16 can differ from direct f64 -> bf16 only
    when the f32 value lands exactly on a bf16 tie; the generator defines its
    values as this two-step rounding, so both sides see the same bits.
    """
    f32 = np.ascontiguousarray(a, dtype=np.float32)
    u = f32.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact float64 value of bf16 bit patterns (bf16 is a subset of f64)."""
    u = bits.astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def bits_to_torch(bits: np.ndarray, device="cpu"):
    """uint16 bf16 bit patterns -> torch.bfloat16 tensor with identical bits."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16))
    return t.view(torch.bfloat16).to(device)


# ---------------------------------------------------------------------------
# random streams
# ---------------------------------------------------------------------------

def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


def _modes(seed: int, stream: int, W: int, n_px_lat: int):
    """M random Fourier modes (integer longitude wavenumbers for periodicity)."""
    g = _rng(seed, 1, stream)
    ell = CORR_TOKENS * PATCH                      # correlation length in pixels
    # squared-exponential spectrum: angular wavenumbers ~ N(0, 1/ell^2)
    wx = g.normal(0.0, 1.0 / ell, N_MODES)
    wy = g.normal(0.0, 1.0 / ell, N_MODES)
    kx = np.round(wx * W / (2 * np.pi))            # cycles around the longitude circle
    phase = g.uniform(0.0, 2 * np.pi, N_MODES)
    return kx, wy, phase


def _fourier(kx, wy, phase, lon_px, lat_px, W, shift_px=0):
    """sum_m sqrt(2/M) cos(2 pi kx_m (lon - shift)/W + wy_m lat + phase_m)."""
    arg = (2 * np.pi / W) * np.multiply.outer(lon_px - shift_px, kx)[None, :, :] \
        + np.multiply.outer(lat_px, wy)[:, None, :] + phase
    return np.sqrt(2.0 / N_MODES) * np.cos(arg).sum(-1)


def _pixel_frame(N: int, seed: int, t: int, static_cache: dict) -> np.ndarray:
    """[2 n_lat, 2 n_lon, C] pixel channels of frame t."""
    n_lat, n_lon = grid_shape(N)
    Hp, W = PATCH * n_lat, PATCH * n_lon
    lat_px = np.arange(Hp, dtype=np.float64)
    lon_px = np.arange(W, dtype=np.float64)
    key = (N, seed)
    if key not in static_cache:
        oro = _fourier(*_modes(seed, 100, W, Hp), lon_px, lat_px, W)
        lsm_src = _fourier(*_modes(seed, 101, W, Hp), lon_px, lat_px, W)
        lsm = np.where(lsm_src > 0.0, 1.0, -1.0)
        lat_deg = 90.0 - (lat_px + 0.5) * (180.0 / Hp)
        lat = np.sqrt(2.0) * np.sin(np.deg2rad(lat_deg))[:, None] * np.ones((1, W))
        static_cache[key] = np.stack([oro, lsm, lat], axis=-1)
    static = static_cache[key]
    dyn = []
    noise = _rng(seed, 2, t).normal(0.0, NOISE_STD, (Hp, W, 3))
    for c in range(3):
        kx, wy, ph = _modes(seed, c, W, Hp)
        dyn.append(_fourier(kx, wy, ph, lon_px, lat_px, W, shift_px=PATCH * t))
    dyn = np.stack(dyn, axis=-1) + noise
    return np.concatenate([static, dyn], axis=-1)


def _patches(px: np.ndarray) -> np.ndarray:
    """[2 n_lat, 2 n_lon, C] -> [N, C*p*p] tokens, lat-major, features (c, py, px)."""
    Hp, W, C = px.shape
    n_lat, n_lon = Hp // PATCH, W // PATCH
    a = px.reshape(n_lat, PATCH, n_lon, PATCH, C).transpose(0, 2, 4, 1, 3)
    return a.reshape(n_lat * n_lon, C * PATCH * PATCH)


def _projection(role: str, H: int, d: int, proj_seed: int) -> np.ndarray:
    F = N_CHANNELS * PATCH * PATCH
    g = _rng(proj_seed, 10 + ROLES[role], H, d)
    return g.normal(0.0, 1.0 / math.sqrt(F), (F, H * d))


def make_field(K: int, N: int, H: int, d: int, seed: int = 0, role: str = "x",
               frames: Optional[Sequence[int]] = None,
               tokens: Optional[slice] = None,
               proj_seed: int = PROJ_SEED, scale: float = 1.0) -> np.ndarray:
    """bf16 bits [len(frames), n_tokens, H, d] of the synthetic field (role x/q/k/v)."""
    frames = range(K) if frames is None else frames
    tokens = slice(0, N) if tokens is None else tokens
    Wp = _projection(role, H, d, proj_seed) * scale
    cache: dict = {}
    out = []
    for t in frames:
        feat = _patches(_pixel_frame(N, seed, t, cache))[tokens]
        y = np.clip(feat @ Wp, -CLIP, CLIP)
        out.append(f64_to_bf16_bits(y).reshape(-1, H, d))
    return np.stack(out, axis=0)


def make_iid(K: int, N: int, H: int, d: int, seed: int = 0, role: str = "x",
             frames: Optional[Sequence[int]] = None, tokens: Optional[slice] = None,
             scale: float = 1.0) -> np.ndarray:
    """bf16 bits of N(0, scale^2) clipped to +-4, keyed per (seed, role, frame)."""
    frames = range(K) if frames is None else frames
    tokens = slice(0, N) if tokens is None else tokens
    out = []
    for t in frames:
        g = _rng(seed, 3, ROLES[role], t)
        a = np.clip(g.normal(0.0, scale, (N, H, d)), -CLIP, CLIP)[tokens]
        out.append(f64_to_bf16_bits(a))
    return np.stack(out, axis=0)


def _make(kind, K, N, H, d, seed, role, frames, tokens, scale):
    if kind == "field":
        return make_field(K, N, H, d, seed, role, frames, tokens, scale=scale)
    if kind == "iid":
        return make_iid(K, N, H, d, seed, role, frames, tokens, scale=scale)
    raise ValueError(f"unknown input kind {kind!r}")


def make_qkv(K, N, H, d, seed=0, kind="field", peaky=False, frames=None, tokens=None):
    """Three independent inputs (q, k, v) for the standalone attention calls.

    peaky=True scales q by 4 before clipping (softmax stress).
    """
    q = _make(kind, K, N, H, d, seed, "q", frames, tokens, 4.0 if peaky else 1.0)
    k = _make(kind, K, N, H, d, seed, "k", frames, tokens, 1.0)
    v = _make(kind, K, N, H, d, seed, "v", frames, tokens, 1.0)
    return q, k, v


def make_x(K, N, H, d, seed=0, kind="field", frames=None, tokens=None):
    """The single block input x (q = k = v = x per stage, reading G1)."""
    return _make(kind, K, N, H, d, seed, "x", frames, tokens, 1.0)


# ---------------------------------------------------------------------------
# random parameters of the full divided block (NEXT-1): draws only
# ---------------------------------------------------------------------------

BLOCK_PARAM_SHAPES = {  # name -> (shape as a function of D = H d and F, kind)
    "ln_t_g": ("D", "gain"), "ln_t_b": ("D", "bias"),
    "w_qkv_t": ("3D,D", "weight"), "b_qkv_t": ("3D", "bias"),
    "w_o_t": ("D,D", "weight"), "b_o_t": ("D", "bias"),
    "ln_s_g": ("D", "gain"), "ln_s_b": ("D", "bias"),
    "w_qkv_s": ("3D,D", "weight"), "b_qkv_s": ("3D", "bias"),
    "w_o_s": ("D,D", "weight"), "b_o_s": ("D", "bias"),
    "ln_m_g": ("D", "gain"), "ln_m_b": ("D", "bias"),
    "w_1": ("F,D", "weight"), "b_1": ("F", "bias"),
    "w_2": ("D,F", "weight"), "b_2": ("D", "bias"),
}


def make_block_params(H: int, d: int, F: int, seed: int = 7) -> dict:
    """Random-init parameters of one divided block (there are no trained weights).

    Weights [out, in] ~ N(0, 1/in) rounded to bf16 (returned as uint16 bits);
    LayerNorm gains 1 + N(0, 0.1^2), biases N(0, 0.1^2), both rounded to fp32
    (returned as float32).  Keyed by (seed, parameter index).
    """
    D = H * d
    dims = {"D": D, "3D": 3 * D, "F": F}
    out = {}
    for i, (name, (shp, kind)) in enumerate(BLOCK_PARAM_SHAPES.items()):
        shape = tuple(dims[s] for s in shp.split(","))
        g = _rng(seed, 50 + i)
        if kind == "weight":
            out[name] = f64_to_bf16_bits(g.normal(0.0, 1.0 / math.sqrt(shape[1]), shape))
        elif kind == "gain":
            out[name] = (1.0 + g.normal(0.0, 0.1, shape)).astype(np.float32)
        else:
            out[name] = g.normal(0.0, 0.1, shape).astype(np.float32)
    return out


def block_params_f64(params: dict) -> dict:
    """The exact float64 values of make_block_params' bf16 / fp32 parameters."""
    return {k: (bf16_bits_to_f64(v) if v.dtype == np.uint16 else v.astype(np.float64)) for k, v in params.items()}
