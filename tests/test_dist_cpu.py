"""Multi-process (world_size 2, gloo, CPU) checks of the distributed path's host logic.

The CUDA path (tsf.cu all_to_all_xt / tsf_reshard) shards temporal attention by
token and spatial attention by frame and moves X_t with one byte-typed
all-to-all: the chunk for peer p is the contiguous frame range
[p K/P, (p+1) K/P) of the local token shard, the receive buffer is
[P][K/P][N/P][H][d] and is unpacked to [K/P][N][H][d].  These tests run that
exact chunk/byte plan across two processes with gloo and check it against
(a) plain slicing of the full tensor and (b) the single-process oracle block.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def plan_t2s(token_shard: np.ndarray, P: int) -> np.ndarray:
    """The byte plan of all_to_all_xt, executed with gloo: -> frame shard."""
    K, Nc, H, d = token_shard.shape
    Kc = K // P
    raw = torch.from_numpy(np.ascontiguousarray(token_shard).view(np.uint8).reshape(-1))
    recv = torch.empty_like(raw)
    dist.all_to_all_single(recv, raw)       # equal contiguous chunks: chunk p = frames of peer p
    blocks = recv.numpy().view(token_shard.dtype).reshape(P, Kc, Nc, H, d)
    return np.concatenate(list(blocks), axis=1)      # unpack [P][Kc][Nc] -> [Kc][P*Nc]


def plan_s2t(frame_shard: np.ndarray, P: int) -> np.ndarray:
    """tsf_reshard(TSF_S2T): pack [Kc][N] -> [P][Kc][Nc], all-to-all, received = [K][Nc]."""
    Kc, N, H, d = frame_shard.shape
    Nc = N // P
    packed = np.ascontiguousarray(frame_shard.reshape(Kc, P, Nc, H, d).transpose(1, 0, 2, 3, 4))
    raw = torch.from_numpy(packed.view(np.uint8).reshape(-1))
    recv = torch.empty_like(raw)
    dist.all_to_all_single(recv, raw)
    return recv.numpy().view(frame_shard.dtype).reshape(P * Kc, Nc, H, d)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.random.default_rng(7)
        K, N, H, d = 4, 6, 2, 4
        x = g.normal(size=(K, N, H, d))                          # same on every rank (seeded)
        xs = oracle.shard_tokens(x, world, rank)
        # bit-exact reshard of arbitrary 16-bit payloads (the kernel moves fp16 X_t as bytes)
        bits = g.integers(0, 2 ** 16, size=(K, N, H, d), dtype=np.uint16)
        fr = plan_t2s(oracle.shard_tokens(bits, world, rank), world)
        ok_t2s = np.array_equal(fr, oracle.shard_frames(bits, world, rank))
        back = plan_s2t(fr, world)
        ok_round = np.array_equal(back, oracle.shard_tokens(bits, world, rank))
        # distributed block = temporal on token shard, reshard, spatial on frame shard
        xt = xs + oracle.temporal(xs, xs, xs)
        xt_fr = plan_t2s(xt, world)
        y = xt_fr + oracle.spatial(xt_fr, xt_fr, xt_fr)
        err = float(np.abs(y - oracle.shard_frames(oracle.block(x), world, rank)).max())
        q.put((rank, ok_t2s, ok_round, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_plan_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_t2s, ok_round, err in res:
        assert ok_t2s, f"rank {rank}: token->frame reshard is not the index permutation"
        assert ok_round, f"rank {rank}: s2t(t2s(x)) != x"
        assert err <= 1e-12, f"rank {rank}: distributed block differs from block by {err}"


def test_divisibility_is_required():
    with pytest.raises(ValueError):
        oracle.shard_tokens(np.zeros((4, 6, 1, 2)), 4, 0)
    with pytest.raises(ValueError):
        oracle.shard_frames(np.zeros((6, 4, 1, 2)), 4, 0)
