"""Benchmark of the factorized space-time attention block (one "step" = one
tsf_spacetime_block over a [K, N, H, d] synthetic field: temporal attention,
[all-to-all], spatial attention, residuals).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tsf|reference]

N = 1: BASELINE.json configs[1] (C2: K=8, N=4096, H=16, d=64).  N > 1 (torchrun,
one process per GPU, NCCL): weak scaling with C2 per GPU, K = 8 * N frames,
x token-sharded in, y frame-sharded out, one all-to-all per step.

Prints ONE JSON line on rank 0 (the driver's contract).
--impl reference times the fp64 CPU oracle on bounded samples of the same
workload (the tier's reference arm) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time tokens/s per attention layer"
UNIT = "tokens/s"
BASE = dict(K=8, N=4096, H=16, d=64)          # BASELINE.json configs[1] (C2)
# --config: the default C2 is weak scaling (K = 8 per GPU); C4 is weak scaling
# with K = 16 per GPU; C3 and C5 are strong scaling (fixed shape).
CONFIGS = {
    "C2": dict(K=8, N=4096, H=16, d=64, weak=True),
    "C3": dict(K=32, N=16384, H=16, d=64, weak=False),
    "C4": dict(K=16, N=65536, H=16, d=128, weak=True),
    "C5": dict(K=1024, N=1024, H=8, d=64, weak=False),
}


def shape_for(cfg, world):
    c = CONFIGS[cfg]
    K = c["K"] * world if c["weak"] else c["K"]
    return K, c["N"], c["H"], c["d"], ("weak" if c["weak"] else "strong")
L2_BYTES = 126 * 2 ** 20


def peaks():
    """MEASURED_PEAKS.json (driver-written), else the profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return dict(tflops=m["bf16_tflops"], tflops_sustained=m.get("bf16_tflops_sustained"),
                    hbm=m["hbm_gbs"], source="MEASURED_PEAKS.json (measured)")
    except Exception:
        return dict(tflops=1590.0, tflops_sustained=1400.0, hbm=6650.0,
                    source="B200_PROFILING.md fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "note": getattr(self, "note", "timed region")}


def traffic_from_profiles(kernel_tag: str):
    """dram bytes per launch of the dominant kernel from a committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel_tag)
    except Exception:
        return None


def cpu_baseline(K, N, H, d, seconds=12.0, label="oracle"):
    """Time the fp64 oracle (as it stands) on host cores: full (t, h) planes of the
    block, i.e. y[t, :, h, :], until about `seconds` of CPU work."""
    import numpy as np
    import oracle
    import synth
    cores = len(os.sched_getaffinity(0))
    frames = list(range(K))
    x = synth.bf16_bits_to_f64(synth.make_x(K, N, H, d, seed=0, frames=frames))
    planes, t0 = 0, time.perf_counter()
    order = [(t, h) for h in range(H) for t in range(K)]
    while True:
        t, h = order[planes % len(order)]
        oracle.block_plane(x, t, h)
        planes += 1
        el = time.perf_counter() - t0
        if el >= seconds or planes >= 4 * len(order):
            break
    tokens = planes * N / H          # a plane is 1/H of the work of N tokens
    return {"value": tokens / el, "unit": UNIT, "cores": cores, "kind": label,
            "sample": f"{planes} full (t,h) planes y[t,:,h,:] of the block at K={K} N={N} H={H} d={d} "
                      f"(= {tokens:.0f} token-equivalents) in {el:.1f} s, numpy fp64, BLAS threads = cores"}


def run_reference(args, rank, world):
    """Reference arm: the fp64 oracle on bounded samples, rank 0 only."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    K, N, H, d = BASE["K"] * world, BASE["N"], BASE["H"], BASE["d"]
    x = synth.bf16_bits_to_f64(synth.make_x(K, N, H, d, seed=0, frames=range(min(K, 8 * world))))
    order = [(t, h) for h in range(H) for t in range(x.shape[0])]
    for i in range(args.warmup):
        oracle.block_plane(x, *order[i % len(order)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.block_plane(x, *order[(args.warmup + i) % len(order)])
    el = time.perf_counter() - t0
    tokens = args.steps * N / H
    value = tokens / el
    cores = len(os.sched_getaffinity(0))
    sample = (f"one full (t,h) plane y[t,:,h,:] of the block per step (N/H = {N // H} token-equivalents), "
              f"K={K} N={N} H={H} d={d}, numpy fp64")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload_config(K, N, H, d, world), l2_sets=l2_sets(K, N, H, d, world)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def l2_sets(K, N, H, d, world):
    """Rotating input/output sets so a step never finds its data in L2 (each set
    is one rank's bf16 x token shard + fp32 y frame shard; R sets > 3x L2)."""
    set_bytes = K * (N // world) * H * d * 2 + (K // world) * N * H * d * 4
    return max(2, -(-3 * L2_BYTES // set_bytes))


def workload_config(K, N, H, d, world, cfg="C2"):
    if cfg == "C2":
        wl = (f"C2 per GPU (BASELINE.json configs[1]): K={K} frames (8 per GPU), N={N} tokens "
              f"(64x64 lat-lon patches), H={H}, d={d}, batch 1; factorized block temporal->spatial")
    else:
        wl = (f"{cfg} (BASELINE.json configs[{'C1 C2 C3 C4 C5'.split().index(cfg)}]): K={K}, N={N}, H={H}, d={d}, "
              f"batch 1; factorized block temporal->spatial; inputs iid N(0,1) clipped to +-4 (device-generated)")
    return {"workload": wl,
            "K": K, "N": N, "H": H, "d": d, "global_batch": 1, "seq_len": K * N,
            "parallelism": f"axis-sharded x{world} (temporal by token, spatial by frame, 1 all-to-all)"
            if world > 1 else "single GPU",
            "l2": "rotating input/output sets larger than L2 (see l2_sets)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="tsf", choices=["tsf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import synth
    import paper_2604_16590_b200 as tsf

    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    K, N, H, d, scaling = shape_for(args.config, world)
    layer = tsf.Layer(K, N, H, d, group=group)
    Nl, Kl = N // world, K // world

    # inputs: this rank's token shard; R rotating sets so a step never finds its
    # input or output in L2 (each set 2*E + 4*E bytes per rank > L2 / R)
    if args.config == "C2":
        xs_bits = synth.make_x(K, N, H, d, seed=0, tokens=slice(rank * Nl, (rank + 1) * Nl))
        x0 = synth.bits_to_torch(xs_bits, "cuda")
    else:  # large shapes: seeded device-side iid inputs (generation is not timed)
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        x0 = torch.randn((K, Nl, H, d), generator=g, device="cuda").clamp_(-4, 4).to(torch.bfloat16)
    R = l2_sets(K, N, H, d, world)
    xs = [x0] + [x0.clone() for _ in range(R - 1)]
    ys = [torch.empty(layer.frame_shard_shape, dtype=torch.float32, device="cuda") for _ in range(R)]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(args.warmup):
        layer.block(xs[i % R], out=ys[i % R])
    torch.cuda.synchronize()
    barrier()

    launches_per_step = layer.last_launch_count()
    layer.set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.steps):
            layer.block(xs[i % R], out=ys[i % R])
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    # per-stage event times of the timed steps only
    st_ms = {s: layer.stage_ms(s) for s in (tsf.STAGE_TEMPORAL, tsf.STAGE_SPATIAL, tsf.STAGE_RESHARD)}
    layer.set_timing(False)
    if world > 1:
        # every rank must run the same number of (collective) steps below
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_all = t.item()
    else:
        ms_all = ms
    if len(clk.lines) < 5:
        # timed region too short for nvidia-smi: sample clocks over a ~1 s
        # repeat of the same step loop (untimed)
        reps = max(1, int(1000.0 / max(ms_all, 1e-3)))
        with ClockSampler(local) as clk:
            for _ in range(reps):
                for i in range(args.steps):
                    layer.block(xs[i % R], out=ys[i % R])
            torch.cuda.synchronize()
        clk.note = f"sampled over a {reps}x repeat of the timed loop"

    # end to end through the C ABI with HOST buffers (pinned), copies timed
    # (two host buffer pairs, alternating).  The headline is the batched call, which
    # pipelines H2D of step i+1 / the block of step i / D2H of step i over the two PCIe
    # directions; one tsf_spacetime_block_host call per step (copies and block
    # serialised) is kept beside it.
    xh = [xs[i % R].cpu().pin_memory() for i in range(2)]
    yh = [torch.empty(layer.frame_shard_shape, dtype=torch.float32).pin_memory() for _ in range(2)]
    e2e_steps = max(3, min(args.steps, 50))
    layer.block_host_batch(xh, yh)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    layer.block_host_batch([xh[i % 2] for i in range(e2e_steps)], [yh[i % 2] for i in range(e2e_steps)])
    barrier()
    e2e_s = time.perf_counter() - t0
    layer.block_host(xh[0], yh[0])
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        layer.block_host(xh[i % 2], yh[i % 2])
    barrier()
    e2e1_s = time.perf_counter() - t0

    # the same temporal kernel writing locally (no exchange): a single-GPU handle of
    # this rank's token-shard shape, timed on its own (fused-exchange bandwidth)
    tl_ms = 0.0
    if world > 1 and layer.exchange_mode() == 2:
        loc = tsf.Layer(K, Nl, H, d)
        yl = torch.empty((K, Nl, H, d), dtype=torch.float32, device="cuda")
        for i in range(3):
            loc.block(xs[i % R], out=yl)
        torch.cuda.synchronize()
        loc.set_timing(True)
        reps = max(20, min(args.steps, 200))
        for i in range(reps):
            loc.block(xs[i % R], out=yl)
        torch.cuda.synchronize()
        tl_ms = loc.stage_ms(tsf.STAGE_TEMPORAL)[0] / reps
        loc.close()
        del yl

    # max over ranks
    vals = torch.tensor([ms, e2e_s, st_ms[1][0], st_ms[0][0], st_ms[2][0], tl_ms, e2e1_s], dtype=torch.float64,
                        device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_s, sp_ms, tp_ms, rs_ms, tl_ms, e2e1_s = vals.tolist()

    if rank == 0:
        pk = peaks()
        tokens = K * N
        step_ms = ms / args.steps
        value = tokens * args.steps / (ms / 1e3)
        F = tsf.flops(K, N, H, d)
        # dominant kernel: the spatial flash-attention kernel; algorithmic flops
        # per step = 4 H d Kl N^2 (QK^T + PV) on this rank, split over the
        # launches of a step (1, or one per head chunk when P > 1)
        n_sp = st_ms[1][1]
        per_step = max(n_sp // args.steps, 1)
        sp_launch_ms = sp_ms / max(n_sp, 1)
        sp_flops = 4 * H * d * Kl * N * N // per_step
        achieved = sp_flops / (sp_launch_ms / 1e3) / 1e12
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16 in; fp16 X_t, MMA operands and P; fp32 accumulate and y",
            "data": "synthetic",
            "config": dict(workload_config(K, N, H, d, world, args.config), l2_sets=R),
            "tflops": F / (step_ms / 1e3) / 1e12,
            "tflops_frac_of_measured": F / (step_ms / 1e3) / 1e12 / (pk["tflops"] * world),
            "roofline": {"bound": "tensor", "kernel": f"attn_flash_kernel<{d}, EPI_BLOCK_S> (spatial stage)",
                         "achieved": achieved, "peak": pk["tflops"], "unit": "TFLOP/s",
                         "frac": achieved / pk["tflops"], "traffic": traffic_from_profiles(f"spatial_{args.config}"),
                         "peak_source": pk["source"] + " bf16 burst (fp16 operands: same nominal rate)",
                         "algorithmic_flops_per_launch": sp_flops, "launch_ms": sp_launch_ms,
                         "launches_per_step": per_step,
                         "stage_ms_per_step": {"temporal": tp_ms / args.steps, "spatial": sp_ms / args.steps,
                                               "exchange (comm stream)": rs_ms / args.steps}},
            "e2e": {"value": tokens * e2e_steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": xh[0].numel() * 2, "d2h_bytes_per_step": yh[0].numel() * 4,
                    "api": f"tsf_spacetime_block_host_batch, {e2e_steps} steps (pinned host buffers, "
                           "H2D / block / D2H pipelined)",
                    "unpipelined_value": tokens * e2e_steps / e2e1_s,
                    "unpipelined_api": "tsf_spacetime_block_host once per step"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        if world > 1:
            a2a_bytes = xs[0].numel() * 2            # X_t (fp16) bytes per rank entering the exchange
            rs_step_ms = rs_ms / args.steps
            fused = layer.exchange_mode() == 2
            line["a2a"] = {"bytes_per_rank": a2a_bytes, "bytes_to_peers_per_rank": a2a_bytes * (world - 1) / world,
                           "ms_per_step_exchange_stage": rs_step_ms, "nvlink_GBs_per_dir": 900}
            if fused:
                line["a2a"]["mode"] = ("fused: the temporal kernel stores X_t rows into each rank's frame shard "
                                       "over NVLink (CUDA IPC); the exchange stage is only the 1-int NCCL "
                                       "all-reduce that orders the stores")
                # exchange bandwidth: the peer stores all happen inside the temporal stage, so
                # bytes to peers / that stage's time is a lower bound of the NVLink rate each
                # rank achieved; the stage's extra time over the same kernel writing locally
                # (P = 1 handle of the rank's token-shard shape) is the exchange's visible cost
                t_ex = tp_ms / args.steps
                to_peers = a2a_bytes * (world - 1) / world
                line["a2a"].update(temporal_ms_local_same_shape=tl_ms, temporal_ms_with_exchange=t_ex,
                                   exchange_visible_ms=t_ex - tl_ms,
                                   nvlink_GBs_per_rank_lower_bound=to_peers / (t_ex / 1e3) / 1e9,
                                   nvlink_frac_lower_bound=to_peers / (t_ex / 1e3) / 1e9 / 900)
            else:
                algbw = a2a_bytes / (rs_step_ms / 1e3) / 1e9
                line["a2a"].update(mode="NCCL grouped send/recv per head chunk; exchange(c+1) overlaps spatial(c)",
                                   algbw_GBs=algbw, busbw_GBs=algbw * (world - 1) / world)
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(min(K, 8), N, H, d)
        print(json.dumps(line), flush=True)
    layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
