"""Timeline of CTA 0 of the flash kernel from clock64 stamps (diagnostics).

    python -m paper_2604_16590_b200.build --trace
    TSF_LIB=paper_2604_16590_b200/libtsf_trace.so python tools/trace_flash.py [K N H d]

Softmax warp stamps per sub-step i: 0 loop top, 1 S ready (s_full), 2 S in
registers, 3 row max done, 4 exponentials done, 5 P stored (after the wait for
PV(G-1)), 6 p_full arrived.  MMA warp (9): per
score tile n = 2i + t: 2n p_full seen, 2n+1 PV(n) and S(n + NB) issued.
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
    what = sys.argv[5] if len(sys.argv) >= 6 else "block"
    layer = tsf.Layer(K, N, H, d)
    x = synth.bits_to_torch(synth.make_iid(K, N, H, d, seed=0), "cuda")
    run = (lambda: layer.block(x)) if what == "block" else (lambda: layer.spatial(x, x, x))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    L = tsf.lib()
    buf = (ctypes.c_ulonglong * (32 * PER_WARP))()
    L.tsf_trace_read.restype = ctypes.c_int
    L.tsf_trace_read(layer._h, buf, 32 * PER_WARP)        # clear
    run()
    torch.cuda.synchronize()
    L.tsf_trace_read(layer._h, buf, 32 * PER_WARP)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(32, PER_WARP).astype(np.int64)
    sub = int(os.environ.get("TSF_SUB", "96" if d == 64 else "128"))
    nsub = (N + sub - 1) // sub
    t0 = a[a > 0].min()
    print(f"{what} TSF_EMU={os.environ.get('TSF_EMU', 'default')} nsub={nsub}  kernel span (CTA0 stamps) {a.max() - t0} cycles")
    phases = ["wait S", "ld S", "max", "exp", "PVwait+st", "arrive", "to next"]
    split = int(os.environ.get("TSF_SPLIT", "1"))
    wmma = 8 * split + 1
    for w in range(8 * split):
        s = a[w, :7 * nsub].reshape(nsub, 7)
        dif = np.diff(s, axis=1)
        nxt = s[1:, 0] - s[:-1, 6]
        per = dif.mean(0).tolist() + [nxt.mean()]
        tot = (s[-1, 6] - s[0, 0]) / nsub
        print(f"warp {w}: cycles/sub-step {tot:7.1f} | " + " ".join(f"{p} {v:6.1f}" for p, v in zip(phases, per)))
    m = a[wmma, :4 * nsub].reshape(2 * nsub, 2)
    print(f"MMA warp {wmma}: mean cycles p_full->issued {np.diff(m, axis=1).mean():.1f}, "
          f"issued->next p_full {(m[1:, 0] - m[:-1, 1]).mean():.1f}")
    print("first sub-steps, warp 0 and warp 4 (relative to kernel start):")
    for i in range(min(6, nsub)):
        print(i, (a[0, 7 * i:7 * i + 7] - t0).tolist(), (a[4 * split, 7 * i:7 * i + 7] - t0).tolist(),
              (a[wmma, 4 * i:4 * i + 4] - t0).tolist())
    # item level (softmax warp 0): item start / last P handed, for up to 256 items
    it = a[0, 512:1024].reshape(256, 2)
    n_it = int(np.count_nonzero(it[:, 0]))
    if n_it > 1:
        dur = np.diff(it[:n_it, 0])
        body = it[:n_it, 1] - it[:n_it, 0]
        print(f"items in CTA0: {n_it}; cycles per item {dur.mean():.0f} = steps {body[:-1].mean():.0f} "
              f"({body[:-1].mean() / nsub:.0f} per step) + epilogue/transition {(dur - body[:-1]).mean():.0f}")
    os.makedirs("gpurun_out", exist_ok=True)
    np.save("gpurun_out/trace_flash.npy", a)


if __name__ == "__main__":
    main()
