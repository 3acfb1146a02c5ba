"""The distributed block (the token->frame exchange) on ONE
GPU: tsf_create_sim runs P virtual ranks with the distributed path's own code
(output routing by frame l -> rank l / (K/P), b_off, per-destination tensor
maps, the flash kernel's staged peer-row epilogue, the NCCL byte plan and the
unpack kernel); only the transport is local.

Bar (BASELINE.json north_star): "the all-to-all reshard must be bit-exact".
  * y of the P-rank block == y of the single-GPU block, bitwise (the
    exchange moves fp16 X_t bytes untouched, and every group is computed by
    the same kernel tile either way);
  * y matches the fp64 oracle on sampled rows within the
    north-star tolerance;
  * tsf_reshard T2S / S2T equal the index permutation of oracle.shard_* (O5).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2


def stack_token_shards(xb, P):
    K, N, H, d = xb.shape
    Nl = N // P
    return np.ascontiguousarray(np.stack([xb[:, r * Nl:(r + 1) * Nl] for r in range(P)]))


def sampled_rows(K, N, H, n, seed):
    g = np.random.default_rng(seed)
    rows = {(int(g.integers(K)), int(g.integers(N)), int(g.integers(H))) for _ in range(n)}
    return sorted(rows | {(0, 0, 0), (K - 1, N - 1, H - 1)})


# (K, N, H, d) per P.  Temporal kernel of each: packed (K <= 128) or flash (K > 128).
def cases():
    out = []
    for P in (2, 4, 8):
        out += [
            pytest.param(P, (8 * P, 4096, 16, 64), id=f"P{P}-C2weak-packed"),    # bench.py --gpus P (weak, C2/GPU)
            pytest.param(P, (200, 8 * P, 2, 64), id=f"P{P}-K200-flash"),         # staged peer rows (flash temporal)
            pytest.param(P, (128, 32 * P, 2, 128), id=f"P{P}-K128-d128"),        # C4-at-P=8 temporal shape
        ]
    out.append(pytest.param(4, (12, 96, 3, 32), id="P4-d32-ragged"))
    # short-window temporal kernel (d = 64, K in {4, 8, 16, 32}) with K/P < 8 frames per
    # rank: its per-destination staging sub-tiles of G * K/P rows (K/P = 4, 2, 1)
    out += [
        pytest.param(2, (8, 256, 2, 64), id="P2-smallt-Kc4"),
        pytest.param(4, (8, 256, 2, 64), id="P4-smallt-Kc2"),
        pytest.param(8, (8, 256, 2, 64), id="P8-smallt-Kc1"),
        pytest.param(4, (16, 128, 3, 64), id="P4-smallt-K16-H3"),
        pytest.param(4, (4, 64, 2, 64), id="P4-smallt-K4-Kc1"),
    ]
    return out


@pytest.fixture(scope="module")
def single_cache():
    return {}


@pytest.mark.parametrize("mode", [2, 1], ids=["fused", "nccl-plan"])
@pytest.mark.parametrize("P,shape", cases())
def test_sim_block_bitwise_equals_single_gpu(tsf_lib, single_cache, P, shape, mode):
    K, N, H, d = shape
    xb = synth.make_x(K, N, H, d, seed=21)
    key = (shape,)
    if key not in single_cache:
        one = tsf_lib.Layer(K, N, H, d)
        single_cache[key] = one.block(synth.bits_to_torch(xb, "cuda")).cpu()
        one.close()
    y1 = single_cache[key]
    sim = tsf_lib.Layer(K, N, H, d, sim_world=P, sim_mode=mode)
    assert sim.exchange_mode() == mode
    xs = synth.bits_to_torch(stack_token_shards(xb, P), "cuda")
    y = sim.block(xs)
    sim.sync()
    y = y.reshape(K, N, H, d).cpu()
    assert torch.equal(y, y1), (f"P={P} mode={mode}: max |dy| = "
                                f"{(y - y1).abs().max().item():.3e} (must be bitwise equal)")
    # oracle parity on sampled rows of the P-rank result itself
    rows = sampled_rows(K, N, H, 96, seed=P)
    want = oracle.block_rows(synth.bf16_bits_to_f64(xb), rows)
    ri = torch.tensor(rows)
    got = y[ri[:, 0], ri[:, 1], ri[:, 2]].double().numpy()
    err = np.abs(got - want)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"P={P} mode={mode} {shape}: max-abs {err.max():.3e} rel-L2 {rel:.3e} max|ref| {np.abs(want).max():.2f}")
    assert err.max() <= MAX_ABS and rel <= REL_L2
    sim.close()


def test_sim_block_host_batch_equals_device_call(tsf_lib):
    """The pipelined host batch on a (simulated) distributed handle: its generic
    branch (whole block, one D2H per item) == the device call, bitwise."""
    K, N, H, d, P = 8, 256, 2, 64, 2
    sim = tsf_lib.Layer(K, N, H, d, sim_world=P)
    xs = [synth.bits_to_torch(stack_token_shards(synth.make_x(K, N, H, d, seed=90 + i), P)) for i in range(3)]
    want = []
    for x in xs:
        want.append(sim.block(x.cuda()).cpu())
    sim.sync()
    yh = [torch.empty(sim.frame_shard_shape, dtype=torch.float32).pin_memory() for _ in xs]
    sim.block_host_batch([x.pin_memory() for x in xs], yh)
    for i in range(3):
        assert torch.equal(yh[i], want[i]), f"item {i}"
    sim.close()


@pytest.mark.parametrize("P,shape", [(2, (8, 64, 2, 64)), (4, (8, 96, 3, 32)), (8, (16, 64, 2, 128))])
def test_sim_reshard_is_the_index_permutation(tsf_lib, P, shape):
    """I10: T2S equals oracle.reshard_t2s of the token shards; S2T o T2S = id (bitwise)."""
    K, N, H, d = shape
    xb = synth.make_x(K, N, H, d, seed=22)
    sim = tsf_lib.Layer(K, N, H, d, sim_world=P, sim_mode=1)
    xs_np = stack_token_shards(xb, P)
    xs = synth.bits_to_torch(xs_np, "cuda")
    fr = sim.reshard(xs, tsf_lib.TSF_T2S)
    back = sim.reshard(fr, tsf_lib.TSF_S2T)
    torch.cuda.synchronize()
    want = oracle.reshard_t2s([xs_np[r] for r in range(P)])
    assert torch.equal(fr.cpu(), synth.bits_to_torch(np.ascontiguousarray(np.stack(want))))
    assert torch.equal(back, xs)
    sim.close()


def test_sim_handle_rejects_bad_world(tsf_lib):
    with pytest.raises(tsf_lib.TsfError) as e:
        tsf_lib.Layer(6, 64, 2, 64, sim_world=4)      # K % P != 0
    assert e.value.status == tsf_lib.TSF_ERR_CONFIG
    with pytest.raises(tsf_lib.TsfError) as e:
        tsf_lib.Layer(8, 64, 2, 64, sim_world=16)     # beyond the 8 GPUs of a box
    assert e.value.status == tsf_lib.TSF_ERR_CONFIG


@pytest.mark.parametrize("P,shape", [(2, (8, 256, 2, 64)), (4, (8, 256, 2, 64)), (4, (200, 16, 2, 64)),
                                     (2, (4, 128, 2, 128))])
def test_sim_block_bwd_equals_single_gpu(tsf_lib, P, shape):
    """NEXT-2, the exchange reversed: the P-rank block backward (dX_t frame shard ->
    token shard as fp32 bytes) matches the single-GPU backward and the fp64 oracle.
    Not bitwise: dq is accumulated with fp32 atomic reductions across key tiles,
    whose order varies (G22); the exchanges themselves are bit-exact
    (test_sim_reshard_is_the_index_permutation)."""
    K, N, H, d = shape
    Nl, Kl = N // P, K // P
    xb = synth.make_x(K, N, H, d, seed=71)
    dy = np.random.default_rng(72).normal(0.0, 1.0, (K, N, H, d)).astype(np.float32)
    one = tsf_lib.Layer(K, N, H, d)
    dx1 = one.block_bwd(synth.bits_to_torch(xb, "cuda"), torch.from_numpy(dy).cuda()).cpu()
    sim = tsf_lib.Layer(K, N, H, d, sim_world=P, sim_mode=1)
    xs = synth.bits_to_torch(stack_token_shards(xb, P), "cuda")
    dys = torch.from_numpy(np.ascontiguousarray(dy)).reshape(P, Kl, N, H, d).cuda()   # frame shards stacked
    dxs = sim.block_bwd(xs, dys)
    sim.sync()
    dx = torch.cat([dxs[r] for r in range(P)], dim=1).cpu()        # token shards -> [K, N, H, d]
    diff = (dx.double() - dx1.double())
    assert diff.norm() <= 1e-4 * dx1.double().norm() and diff.abs().max() <= 1e-2 * dx1.abs().max(), \
        f"P={P}: max |ddx| {diff.abs().max().item():.3e}"
    want = oracle.block_bwd(synth.bf16_bits_to_f64(xb), dy.astype(np.float64))
    rel = np.linalg.norm(dx.double().numpy() - want) / np.linalg.norm(want)
    assert rel <= 2e-2
    one.close()
    sim.close()


def test_stage_bwd_on_a_shard_handle(tsf_lib):
    """The stage backward calls on a (simulated) distributed handle act on one shard."""
    K, N, H, d, P = 8, 256, 2, 64, 4
    sim = tsf_lib.Layer(K, N, H, d, sim_world=P)
    one = tsf_lib.Layer(K // P, N, H, d)
    q, k, v, do = (synth.bits_to_torch(synth.make_iid(K // P, N, H, d, seed=s), "cuda") for s in (81, 82, 83, 84))
    a = sim.attn_bwd(1, q, k, v, do)
    b = one.attn_bwd(1, q, k, v, do)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert (x.float() - y.float()).abs().max().item() <= 1e-2 * y.float().abs().max().item()
