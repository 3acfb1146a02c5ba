"""Summarise a gpurun_out/<tag>/ profiling call into profiles/<tag>/.

    python tools/ncu_summary.py <tag>

Reads gpurun_out/<tag>/{prof.ncu-rep, launches.csv, bench.json} (written by
tools/profile_round.sh on the B200) and writes:
  profiles/<tag>/ncu_full.csv      key metrics per captured kernel (ncu --set full)
  profiles/<tag>/launches.csv      the ncu launch list (cold-cache, serialised)
  profiles/<tag>/SUMMARY.md        tables: metrics, launch shares, bench line
  profiles/traffic.json            dram bytes per launch of the dominant kernels (read by bench.py)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val) * mult


def main(tag, dst_name=None):
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles", dst_name or tag)
    os.makedirs(dst, exist_ok=True)
    md = [f"# Profile {tag}\n"]
    bench_path = os.path.join(src, "bench.json")
    if os.path.exists(bench_path):
        shutil.copy(bench_path, os.path.join(dst, "bench.json"))
        md.append("## bench.py line (plain run, not under ncu)\n\n```\n" + open(bench_path).read().strip() + "\n```\n")
    traffic = {}
    import glob
    reps = sorted(glob.glob(os.path.join(src, "*.ncu-rep")))
    out = []
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            rec = {"kernel": d.get("Kernel Name", "")[:100]}
            for k in KEYS:
                if k in d:
                    rec[k] = d[k] + (f" {u[k]}" if u.get(k) else "")
            rb = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
            wb = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            rec["dram_bytes_per_launch"] = rb + wb
            out.append(rec)
            tag_k = "spatial_C2" if "flash" in rec["kernel"] else "temporal_C2"
            traffic[tag_k] = rb + wb
    if out:
        with open(os.path.join(dst, "ncu_full.csv"), "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(out[0].keys()))
            w.writeheader()
            w.writerows(out)
        md.append("## ncu --set full (one launch each)\n")
        for rec in out:
            md.append(f"### {rec['kernel']}\n")
            for k, v in rec.items():
                if k != "kernel":
                    md.append(f"- `{k}`: {v}")
            md.append("")
    lpath = os.path.join(src, "launches.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(dst, "launches.csv"))
        lines = open(lpath).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
        tot, per = 0.0, {}
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0][:80]
            v = float(r["Metric Value"].replace(",", ""))
            per.setdefault(name, []).append(v)
            tot += v
        md.append("## Launch list (ncu gpu__time_duration, cold cache, serialised)\n")
        md.append("| kernel | launches | mean (ns) | share of listed time |\n|---|---|---|---|")
        for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{name}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.1%} |")
        md.append("")
    with open(os.path.join(dst, "SUMMARY.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    if traffic:
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        cur.update(traffic)
        cur["_source"] = f"profiles/{tag}/ncu_full.csv (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        json.dump(cur, open(tp, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
