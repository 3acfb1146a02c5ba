"""Throughput of the NEXT rows on one GPU, CUDA-event timed:

  * joint attention over all K*N tokens (tsf_joint_attn, the O((KN)^2) regime of
    PAPER.md Table I/II) next to the factorized block at the same shape
  * STORM noise-gated attention (tsf_storm_attn)
  * the full divided block with projections / LN / MLP (tsf_full_block)
  * the backward of the block and of one spatial stage (tsf_*_bwd)

    python tools/bench_next.py [--config C2] [--reps 20]

Prints one JSON line per measurement (numbers from a run under ncu are not
measurements).  Inputs are larger than L2 or rotated (two sets).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_2604_16590_b200 as tsf


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--F", type=int, default=4)
    args = ap.parse_args()
    K, N, H, d = 8, 4096, 16, 64     # C2 (BASELINE.json configs[1])
    D = H * d
    g = torch.Generator(device="cuda").manual_seed(0)
    rnd = lambda *s: torch.randn(*s, generator=g, device="cuda").clamp_(-4, 4).to(torch.bfloat16)
    xs = [rnd(K, N, H, d) for _ in range(2)]
    layer = tsf.Layer(K, N, H, d)
    out = {}
    # factorized block vs joint attention at C2
    ms_block = timed(lambda i: layer.block(xs[i % 2]), args.reps)
    F_block = tsf.flops(K, N, H, d)
    out["factorized_block"] = {"ms": ms_block, "tokens_per_s": K * N / ms_block * 1e3,
                               "tflops": F_block / ms_block / 1e9}
    for mask, name in ((0, "joint_unmasked"), (3, "joint_causal_frames")):
        ms = timed(lambda i: layer.joint(xs[i % 2], xs[i % 2], xs[i % 2], mask=mask), max(3, args.reps // 4))
        L = K * N
        F = 4 * H * d * L * L
        out[name] = {"ms": ms, "tokens_per_s": L / ms * 1e3, "tflops_all_scores": F / ms / 1e9,
                     "vs_factorized_time": ms / ms_block}
    # STORM at C2's frame size: B = 8 states of N = 4096 tokens, M = 256 context tokens
    ctx = [rnd(K, 256, H, d) for _ in range(2)]
    ms = timed(lambda i: layer.storm(xs[i % 2], ctx[i % 2], 1.0, 1.0), args.reps)
    F_storm = 4 * H * d * K * (N * N + N * 256)
    out["storm_attention"] = {"ms": ms, "tokens_per_s": K * N / ms * 1e3, "tflops": F_storm / ms / 1e9,
                              "shape": "B=8 states x N=4096 tokens, M=256 context tokens, H=16, d=64"}
    # full divided block at C2, F = 4 D
    Fh = args.F * D
    params = synth.make_block_params(H, d, Fh, seed=1)
    w = {k: (synth.bits_to_torch(v, "cuda") if v.dtype == np.uint16 else torch.from_numpy(v).cuda())
         for k, v in params.items()}
    layer.set_timing(True)
    ms = timed(lambda i: layer.full_block(xs[i % 2], w), args.reps)
    gemm_ms = layer.stage_ms(7)
    layer.set_timing(False)
    T = K * N
    F_gemm = 2 * T * D * (3 * D + D) * 2 + 2 * T * D * Fh * 2
    out["full_block"] = {"ms": ms, "tokens_per_s": T / ms * 1e3, "F": Fh,
                         "gemm_flops": F_gemm, "attention_flops": F_block,
                         "tflops_total": (F_gemm + F_block) / ms / 1e9,
                         "gemm_and_ln_ms_per_step": gemm_ms[0] / (args.reps + 3)}
    # backward of the block at C2 (NEXT-2): algorithmic flops 2.5x the forward's
    # attention flops (dV, dP, dQ, dK and S^T recompute: 5 matmuls vs 2), the
    # forward recompute with row statistics is inside the timed call
    dy = [torch.randn(K, N, H, d, generator=g, device="cuda") for _ in range(2)]
    ms = timed(lambda i: layer.block_bwd(xs[i % 2], dy[i % 2]), max(3, args.reps // 2))
    out["block_backward"] = {"ms": ms, "tokens_per_s": K * N / ms * 1e3, "flops_bwd_2p5x": 2.5 * F_block,
                             "tflops_bwd_2p5x": 2.5 * F_block / ms / 1e9}
    q3 = [rnd(K, N, H, d) for _ in range(3)]
    ms = timed(lambda i: layer.attn_bwd(1, q3[0], q3[1], q3[2], q3[i % 2]), max(3, args.reps // 2))
    F_sp = 4 * H * d * K * N * N
    out["spatial_attn_backward"] = {"ms": ms, "tflops_bwd_2p5x": 2.5 * F_sp / ms / 1e9,
                                    "note": "includes the forward recompute (row statistics) and dq fp32->bf16"}
    for k, v in out.items():
        print(json.dumps({"what": k, **v}), flush=True)


if __name__ == "__main__":
    main()
