"""Run one parity case on the GPU and print its errors (diagnostics, not a test).

    python tools/gpu_debug.py temporal K N H d [kind]
    python tools/gpu_debug.py spatial  K N H d [kind]
    python tools/gpu_debug.py block    K N H d
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
import synth
import paper_2604_16590_b200 as tsf


def main():
    what = sys.argv[1]
    K, N, H, d = (int(a) for a in sys.argv[2:6])
    kind = sys.argv[6] if len(sys.argv) > 6 else "field"
    layer = tsf.Layer(K, N, H, d)
    t0 = time.time()
    if what == "block":
        xb = synth.make_x(K, N, H, d, seed=0, kind=kind)
        y = layer.block(synth.bits_to_torch(xb, "cuda"))
        torch.cuda.synchronize()
        got = y.double().cpu().numpy()
        want = oracle.block(synth.bf16_bits_to_f64(xb))
    else:
        qb, kb, vb = synth.make_qkv(K, N, H, d, seed=0, kind=kind)
        q, k, v = (synth.bits_to_torch(a, "cuda") for a in (qb, kb, vb))
        o = (layer.temporal if what == "temporal" else layer.spatial)(q, k, v)
        torch.cuda.synchronize()
        got = o.double().cpu().numpy()
        f = oracle.temporal if what == "temporal" else oracle.spatial
        want = f(*(synth.bf16_bits_to_f64(a) for a in (qb, kb, vb)))
    err = np.abs(got - want)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    bad = np.argwhere(err > 2e-2)
    print(f"{what} {K}x{N}x{H}x{d} {kind}: max-abs {err.max():.3e} rel-L2 {rel:.3e} "
          f"nonfinite {np.sum(~np.isfinite(got))} bad {len(bad)} ({time.time() - t0:.1f}s)")
    if len(bad):
        for idx in bad[:6]:
            t, n, h, e = idx
            print("   bad at", tuple(idx), "got", got[t, n, h, e], "want", want[t, n, h, e])
        # which (t, n, h) rows are bad
        rows = {tuple(i[:3]) for i in bad}
        print("   bad rows:", len(rows), sorted(rows)[:10])


if __name__ == "__main__":
    main()
