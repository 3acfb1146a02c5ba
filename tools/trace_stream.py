"""Timeline of CTA 0 of the streaming temporal kernel (attn_stream.cuh), diagnostics.

    python -m paper_2604_16590_b200.build --trace
    TSF_LIB=paper_2604_16590_b200/libtsf_trace.so python tools/trace_stream.py [K N H d]

Stamps (clock64, CTA 0): producer warp 8: stage free (per tile); converter
warp 11: tile landed / converted; QK warp 9 and PV warp 10: operands ready;
softmax warp 0: S ready / P computed / slot free / P handed over; epilogue
warp 4: O ready / O read / staging written / store issued.
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
    nt = int(np.count_nonzero(a[9]))
    t0 = a[a > 0].min()
    r = lambda v: (v - t0).tolist()
    print(f"tiles in CTA0: {nt}")
    print("producer stage-free  :", r(a[8, :nt]))
    print("converter landed     :", r(a[11, 0:2 * nt:2]))
    print("converter done       :", r(a[11, 1:2 * nt:2]))
    print("QK issue             :", r(a[9, :nt]))
    sm = a[0, :4 * nt].reshape(nt, 4)
    print("softmax S ready      :", r(sm[:, 0]))
    print("softmax P computed   :", r(sm[:, 1]))
    print("softmax slot free    :", r(sm[:, 2]))
    print("softmax P handed     :", r(sm[:, 3]))
    print("PV issue             :", r(a[10, :nt]))
    ep = a[4, :4 * nt].reshape(nt, 4)
    print("epilogue O ready     :", r(ep[:, 0]))
    print("epilogue O read      :", r(ep[:, 1]))
    print("epilogue staged      :", r(ep[:, 2]))
    print("epilogue store issued:", r(ep[:, 3]))
    span = ep[-1, 3] - t0
    print(f"span {span} cycles, {span / nt:.0f} per tile; mean softmax {np.mean(sm[:, 3] - sm[:, 0]):.0f}, "
          f"epilogue {np.mean(ep[:, 3] - ep[:, 0]):.0f}, convert {np.mean(a[11, 1:2 * nt:2] - a[11, 0:2 * nt:2]):.0f}")


if __name__ == "__main__":
    main()
