"""B200-native factorized (divided) space-time attention -- Python binding.

Thin ctypes binding over libtsf.so (C ABI in include/tsf.h).  Argument
marshalling only: every step of the path runs in the library's sm_100a
kernels; PyTorch provides device memory, streams and process groups.  There is
no CPU fallback: if libtsf.so is missing or the device is not a B200 the calls
raise.

    import paper_2604_16590_b200 as tsf
    layer = tsf.Layer(K, N, H, d)            # single GPU
    y = layer.block(x)                       # x: bf16 [K, N, H, d] -> y: fp32
    o = layer.temporal(q, k, v); o = layer.spatial(q, k, v)

Distributed (one process per GPU, torch.distributed initialised):
    layer = tsf.Layer(K, N, H, d, group=torch.distributed.group.WORLD)
    y_frames = layer.block(x_tokens)         # [K, N/P, H, d] -> [K/P, N, H, d]
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSF_LIB") or os.path.join(_HERE, "libtsf.so")

# status codes (include/tsf.h)
TSF_OK, TSF_ERR_CONFIG, TSF_ERR_NUMERIC, TSF_ERR_UNSUPPORTED, TSF_ERR_CUDA, TSF_ERR_NCCL, TSF_ERR_NOMEM = \
    0, 2, 3, 4, 5, 6, 7
STATUS_NAMES = {0: "TSF_OK", 2: "TSF_ERR_CONFIG", 3: "TSF_ERR_NUMERIC", 4: "TSF_ERR_UNSUPPORTED",
                5: "TSF_ERR_CUDA", 6: "TSF_ERR_NCCL", 7: "TSF_ERR_NOMEM"}
TSF_T2S, TSF_S2T = 0, 1
TSF_MASK_NONE, TSF_MASK_TEMPORAL, TSF_MASK_SPATIAL, TSF_MASK_CAUSAL_FRAMES = 0, 1, 2, 3
STAGE_TEMPORAL, STAGE_SPATIAL, STAGE_RESHARD, STAGE_COPY, STAGE_TRANSPOSE, STAGE_JOINT, STAGE_STORM = \
    0, 1, 2, 3, 4, 5, 6

# Every function declared in include/tsf.h: (name, restype, argtypes)
_P, _I, _F = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
SIGNATURES = [
    ("tsf_create", _I, [_I, _I, _I, _I, ctypes.POINTER(_P)]),
    ("tsf_temporal_attn", _I, [_P, _P, _P, _P, _P, _P]),
    ("tsf_spatial_attn", _I, [_P, _P, _P, _P, _P, _P]),
    ("tsf_joint_attn", _I, [_P, _P, _P, _P, _P, _I, _P]),
    ("tsf_storm_attn", _I, [_P, _P, _P, _I, ctypes.c_double, ctypes.c_double, _P, _P]),
    ("tsf_full_block", _I, [_P, _P, _P, _P, _P]),
    ("tsf_temporal_attn_bwd", _I, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("tsf_spatial_attn_bwd", _I, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("tsf_spacetime_block_bwd", _I, [_P, _P, _P, _P, _P]),
    ("tsf_spacetime_block", _I, [_P, _P, _P, _P]),
    ("tsf_spacetime_block_host", _I, [_P, _P, _P, _P]),
    ("tsf_spacetime_block_host_batch", _I, [_P, _P, _P, _I, _P]),
    ("tsf_destroy", None, [_P]),
    ("tsf_get_unique_id", _I, [_P]),
    ("tsf_create_dist", _I, [_I, _I, _I, _I, _P, _I, _I, ctypes.POINTER(_P)]),
    ("tsf_create_sim", _I, [_I, _I, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    ("tsf_sync", _I, [_P, _P, _I]),
    ("tsf_world_size", _I, [_P]),
    ("tsf_reshard", _I, [_P, _I, _P, _P, _P]),
    ("tsf_transpose", _I, [_P, _I, _I, _P, _P, _P]),
    ("tsf_last_error", ctypes.c_char_p, [_P]),
    ("tsf_last_launch_count", _I, [_P]),
    ("tsf_exchange_mode", _I, [_P]),
    ("tsf_set_timing", _I, [_P, _I]),
    ("tsf_stage_ms", _I, [_P, _I, ctypes.POINTER(_F), ctypes.POINTER(_I)]),
]

_lib = None


BLOCK_WEIGHT_FIELDS = ["ln_t_g", "ln_t_b", "w_qkv_t", "b_qkv_t", "w_o_t", "b_o_t",
                       "ln_s_g", "ln_s_b", "w_qkv_s", "b_qkv_s", "w_o_s", "b_o_s",
                       "ln_m_g", "ln_m_b", "w_1", "b_1", "w_2", "b_2"]


class BlockWeights(ctypes.Structure):
    """tsf_block_weights (include/tsf.h): device pointers + the MLP width F."""
    _fields_ = [(n, ctypes.c_void_p) for n in BLOCK_WEIGHT_FIELDS] + [("F", ctypes.c_int)]


class TsfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libtsf.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2604_16590_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, handle=None):
    if status != TSF_OK:
        msg = lib().tsf_last_error(handle)
        raise TsfError(status, msg.decode() if msg else "")


def _stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _need(t, dtype, shape, name):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


class Layer:
    """One factorized space-time attention layer of shape [K, N, H, d].

    group: a torch.distributed process group for the multi-GPU path (one
    process per GPU); None = single GPU.
    """

    def __init__(self, K: int, N: int, H: int, d: int, group=None, sim_world: int = 0, sim_mode: int = 2):
        self.K, self.N, self.H, self.d = K, N, H, d
        self._h = ctypes.c_void_p()
        self.sim = sim_world > 0
        L = lib()
        if self.sim:
            # one-GPU simulation of sim_world ranks (tsf_create_sim): the calls take
            # every virtual rank's shard stacked on a leading axis
            self.world, self.rank = sim_world, 0
            _check(L.tsf_create_sim(K, N, H, d, sim_world, sim_mode, ctypes.byref(self._h)))
        elif group is None:
            self.world, self.rank = 1, 0
            _check(L.tsf_create(K, N, H, d, ctypes.byref(self._h)))
        else:
            import torch
            import torch.distributed as dist
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
            uid = (ctypes.c_char * 128)()
            if self.rank == 0:
                _check(L.tsf_get_unique_id(uid))
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=dist.get_global_rank(group, 0), group=group)
            raw = bytes(t.cpu().tolist())
            uid = (ctypes.c_char * 128).from_buffer_copy(raw)
            _check(L.tsf_create_dist(K, N, H, d, uid, self.rank, self.world, ctypes.byref(self._h)))

    # shapes of the shards this rank holds (a simulated handle: all ranks' shards stacked)
    @property
    def token_shard_shape(self):
        s = (self.K, self.N // self.world, self.H, self.d)
        return (self.world,) + s if self.sim else s

    @property
    def frame_shard_shape(self):
        s = (self.K // self.world, self.N, self.H, self.d)
        return (self.world,) + s if self.sim else s

    def close(self):
        if self._h:
            lib().tsf_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- compute ----
    def temporal(self, q, k, v, out=None, stream=None):
        """tsf_temporal_attn: q, k, v bf16 [K, N/P, H, d] -> bf16 (P:64 temporal)."""
        import torch
        shp = self.token_shard_shape[-4:]
        for t, n in ((q, "q"), (k, "k"), (v, "v")):
            _need(t, torch.bfloat16, shp, n)
        out = torch.empty_like(q) if out is None else out
        _need(out, torch.bfloat16, shp, "out")
        _check(lib().tsf_temporal_attn(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                       _stream_ptr(stream)), self._h)
        return out

    def spatial(self, q, k, v, out=None, stream=None):
        """tsf_spatial_attn: q, k, v bf16 [K/P, N, H, d] -> bf16 (P:64 spatial)."""
        import torch
        shp = self.frame_shard_shape[-4:]
        for t, n in ((q, "q"), (k, "k"), (v, "v")):
            _need(t, torch.bfloat16, shp, n)
        out = torch.empty_like(q) if out is None else out
        _need(out, torch.bfloat16, shp, "out")
        _check(lib().tsf_spatial_attn(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                      _stream_ptr(stream)), self._h)
        return out

    def joint(self, q, k, v, mask: int = TSF_MASK_NONE, out=None, stream=None):
        """tsf_joint_attn: global attention over all K*N tokens (bf16 [K, N, H, d]), O((KN)^2),
        with an optional TSF_MASK_* (temporal / spatial block mask, causal frames)."""
        import torch
        shp = (self.K, self.N, self.H, self.d)
        for t, n in ((q, "q"), (k, "k"), (v, "v")):
            _need(t, torch.bfloat16, shp, n)
        out = torch.empty_like(q) if out is None else out
        _need(out, torch.bfloat16, shp, "out")
        _check(lib().tsf_joint_attn(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), int(mask),
                                    _stream_ptr(stream)), self._h)
        return out

    def storm(self, u, ctx, sigma: float, sigma_data: float, out=None, stream=None):
        """tsf_storm_attn: y = u + (1-g) SelfAttn(u) + g CrossAttn(u, ctx), g = s^2/(s^2 + s_data^2).
        u bf16 [K, N, H, d] (K independent states), ctx bf16 [K, M, H, d] -> y fp32 [K, N, H, d]."""
        import torch
        _need(u, torch.bfloat16, (self.K, self.N, self.H, self.d), "u")
        if ctx.dim() != 4 or tuple(ctx.shape[::2]) != (self.K, self.H) or ctx.shape[3] != self.d:
            raise ValueError(f"ctx must have shape ({self.K}, M, {self.H}, {self.d}), got {tuple(ctx.shape)}")
        _need(ctx, torch.bfloat16, tuple(ctx.shape), "ctx")
        out = torch.empty((self.K, self.N, self.H, self.d), dtype=torch.float32, device=u.device) \
            if out is None else out
        _need(out, torch.float32, (self.K, self.N, self.H, self.d), "out")
        _check(lib().tsf_storm_attn(self._h, u.data_ptr(), ctx.data_ptr(), int(ctx.shape[1]), float(sigma),
                                    float(sigma_data), out.data_ptr(), _stream_ptr(stream)), self._h)
        return out

    def full_block(self, x, weights: dict, out=None, stream=None):
        """tsf_full_block: the full divided block (pre-LN, QKV / O projections, MLP) around
        the factorized attention.  weights: name -> CUDA tensor (bf16 [out, in] weights,
        fp32 vectors), names as in BLOCK_WEIGHT_FIELDS.  x bf16 [K, N, H, d] -> y fp32."""
        import torch
        shp = (self.K, self.N, self.H, self.d)
        _need(x, torch.bfloat16, shp, "x")
        D = self.H * self.d
        F = weights["w_1"].shape[0]
        want = {"w_qkv_t": (3 * D, D), "w_o_t": (D, D), "w_qkv_s": (3 * D, D), "w_o_s": (D, D),
                "w_1": (F, D), "w_2": (D, F), "b_qkv_t": (3 * D,), "b_qkv_s": (3 * D,), "b_1": (F,)}
        st = BlockWeights()
        for n in BLOCK_WEIGHT_FIELDS:
            t = weights[n]
            _need(t, torch.bfloat16 if n.startswith("w_") else torch.float32, want.get(n, (D,)), n)
            if not t.is_cuda:
                raise ValueError(f"{n} must be a CUDA tensor")
            setattr(st, n, t.data_ptr())
        st.F = F
        out = torch.empty(shp, dtype=torch.float32, device=x.device) if out is None else out
        _need(out, torch.float32, shp, "out")
        _check(lib().tsf_full_block(self._h, ctypes.byref(st), x.data_ptr(), out.data_ptr(), _stream_ptr(stream)),
               self._h)
        return out

    def attn_bwd(self, axis: int, q, k, v, dO, stream=None):
        """tsf_temporal_attn_bwd (axis 0) / tsf_spatial_attn_bwd (axis 1): (dq, dk, dv) bf16."""
        import torch
        shp = (self.token_shard_shape if axis == 0 else self.frame_shard_shape)[-4:]
        for t, n in ((q, "q"), (k, "k"), (v, "v"), (dO, "dO")):
            _need(t, torch.bfloat16, shp, n)
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        fn = lib().tsf_temporal_attn_bwd if axis == 0 else lib().tsf_spatial_attn_bwd
        _check(fn(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), dO.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                  dv.data_ptr(), _stream_ptr(stream)), self._h)
        return dq, dk, dv

    def block_bwd(self, x, dy, out=None, stream=None):
        """tsf_spacetime_block_bwd: x bf16 (token shard), dy fp32 (frame shard) -> dx fp32
        (token shard); all [K, N, H, d] on one GPU.  Distributed / simulated handles run
        the exchange reversed (frame -> token shard for dX_t)."""
        import torch
        _need(x, torch.bfloat16, self.token_shard_shape, "x")
        _need(dy, torch.float32, self.frame_shard_shape, "dy")
        out = torch.empty(self.token_shard_shape, dtype=torch.float32, device=x.device) if out is None else out
        _need(out, torch.float32, self.token_shard_shape, "out")
        _check(lib().tsf_spacetime_block_bwd(self._h, x.data_ptr(), dy.data_ptr(), out.data_ptr(), _stream_ptr(stream)),
               self._h)
        return out

    def block(self, x, out=None, stream=None):
        """tsf_spacetime_block: x bf16 token shard -> y fp32 frame shard."""
        import torch
        _need(x, torch.bfloat16, self.token_shard_shape, "x")
        out = torch.empty(self.frame_shard_shape, dtype=torch.float32, device=x.device) if out is None else out
        _need(out, torch.float32, self.frame_shard_shape, "out")
        _check(lib().tsf_spacetime_block(self._h, x.data_ptr(), out.data_ptr(), _stream_ptr(stream)), self._h)
        return out

    def block_host(self, x_host, y_host, stream=None):
        """tsf_spacetime_block_host: CPU (pinned) bf16 x -> CPU fp32 y, copies included."""
        import torch
        _need(x_host, torch.bfloat16, self.token_shard_shape, "x_host")
        _need(y_host, torch.float32, self.frame_shard_shape, "y_host")
        if x_host.is_cuda or y_host.is_cuda:
            raise ValueError("block_host takes host tensors")
        _check(lib().tsf_spacetime_block_host(self._h, x_host.data_ptr(), y_host.data_ptr(), _stream_ptr(stream)),
               self._h)
        return y_host

    def block_host_batch(self, xs_host, ys_host, stream=None):
        """tsf_spacetime_block_host_batch: lists of CPU (pinned) bf16 x / fp32 y tensors,
        n independent blocks with H2D, compute and D2H pipelined."""
        import torch
        if len(xs_host) != len(ys_host):
            raise ValueError("xs_host and ys_host differ in length")
        for x, y in zip(xs_host, ys_host):
            _need(x, torch.bfloat16, self.token_shard_shape, "x_host")
            _need(y, torch.float32, self.frame_shard_shape, "y_host")
            if x.is_cuda or y.is_cuda:
                raise ValueError("block_host_batch takes host tensors")
        n = len(xs_host)
        xa = (_P * max(n, 1))(*[x.data_ptr() for x in xs_host])
        ya = (_P * max(n, 1))(*[y.data_ptr() for y in ys_host])
        _check(lib().tsf_spacetime_block_host_batch(self._h, xa, ya, n, _stream_ptr(stream)), self._h)
        return ys_host

    def reshard(self, x, direction: int, out=None, stream=None):
        """tsf_reshard: TSF_T2S token shard -> frame shard, TSF_S2T the inverse (bit-exact)."""
        import torch
        src, dst = ((self.token_shard_shape, self.frame_shard_shape) if direction == TSF_T2S
                    else (self.frame_shard_shape, self.token_shard_shape))
        _need(x, torch.bfloat16, src, "x")
        out = torch.empty(dst, dtype=torch.bfloat16, device=x.device) if out is None else out
        _need(out, torch.bfloat16, dst, "out")
        _check(lib().tsf_reshard(self._h, direction, x.data_ptr(), out.data_ptr(), _stream_ptr(stream)), self._h)
        return out

    def transpose(self, x, out=None, stream=None):
        """tsf_transpose: bf16 [A, B, H, d] -> [B, A, H, d] (frame-major <-> token-major)."""
        import torch
        A, B = x.shape[0], x.shape[1]
        _need(x, torch.bfloat16, (A, B, self.H, self.d), "x")
        out = torch.empty((B, A, self.H, self.d), dtype=torch.bfloat16, device=x.device) if out is None else out
        _need(out, torch.bfloat16, (B, A, self.H, self.d), "out")
        _check(lib().tsf_transpose(self._h, A, B, x.data_ptr(), out.data_ptr(), _stream_ptr(stream)), self._h)
        return out

    def sync(self, stream=None, timeout_ms: int = 0):
        """tsf_sync: wait for the stream; raises TsfError(TSF_ERR_NUMERIC) if a block stored a
        non-finite X_t, TsfError(TSF_ERR_NCCL) on an NCCL error or timeout (communicator aborted)."""
        _check(lib().tsf_sync(self._h, _stream_ptr(stream), int(timeout_ms)), self._h)

    # ---- accounting ----
    def last_launch_count(self) -> int:
        return lib().tsf_last_launch_count(self._h)

    def exchange_mode(self) -> int:
        """0 single GPU, 1 NCCL send/recv + unpack, 2 fused NVLink scatter."""
        return lib().tsf_exchange_mode(self._h)

    def set_timing(self, enable: bool):
        _check(lib().tsf_set_timing(self._h, 1 if enable else 0), self._h)

    def stage_ms(self, stage: int):
        ms, n = ctypes.c_float(), ctypes.c_int()
        _check(lib().tsf_stage_ms(self._h, stage, ctypes.byref(ms), ctypes.byref(n)), self._h)
        return ms.value, n.value


def flops(K: int, N: int, H: int, d: int) -> int:
    """Algorithmic flops of one layer: 4 H d (K N^2 + N K^2) (QK^T + PV)."""
    return 4 * H * d * (K * N * N + N * K * K)
