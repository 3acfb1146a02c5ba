"""Timeline of CTA 0 of the packed (short-sequence) kernel (diagnostics).

    TSF_LIB=paper_2604_16590_b200/libtsf_trace.so python tools/trace_packed.py [K N H d]

Softmax warp stamps per tile i: 0 top, 1 S ready, 2 P handed to MMA,
3 next tile converted, 4 O ready, 5 epilogue done.  Trace slots 16+warp.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_2604_16590_b200 as tsf

PER_WARP = 1024


def main():
    K, N, H, d = (int(a) for a in sys.argv[1:5]) if len(sys.argv) >= 5 else (8, 4096, 16, 64)
    layer = tsf.Layer(K, N, H, d)
    x = synth.bits_to_torch(synth.make_iid(K, N, H, d, seed=0), "cuda")
    for _ in range(3):
        layer.block(x)
    torch.cuda.synchronize()
    L = tsf.lib()
    n = 32 * PER_WARP
    buf = (ctypes.c_ulonglong * n)()
    L.tsf_trace_read.restype = ctypes.c_int
    L.tsf_trace_read(layer._h, buf, n)
    layer.block(x)
    torch.cuda.synchronize()
    L.tsf_trace_read(layer._h, buf, n)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(32, PER_WARP).astype(np.int64)
    w0 = a[16]
    ntile = int(np.count_nonzero(w0) // 6)
    s = w0[:6 * ntile].reshape(ntile, 6)
    t0 = s[0, 0]
    print(f"tiles in CTA0: {ntile}, span {s[-1, 5] - t0} cycles, {(s[-1, 5] - t0) / ntile:.0f} per tile")
    names = ["wait S", "softmax+P", "convert next", "wait O", "epilogue", "to next"]
    d = np.diff(s, axis=1)
    nxt = s[1:, 0] - s[:-1, 5]
    print(" | ".join(f"{nm} {v:.0f}" for nm, v in zip(names, list(d.mean(0)) + [nxt.mean()])))
    tma = a[20][:2 * ntile:2]
    mma = a[21][:4 * ntile].reshape(ntile, 4)
    print("TMA issue times (rel):", (tma[:8] - t0).tolist())
    print("MMA S issued / PV issued (rel):", (mma[:6, :2] - t0).tolist())
    print("softmax warp0 tiles (rel):", (s[:6] - t0).tolist())


if __name__ == "__main__":
    main()
