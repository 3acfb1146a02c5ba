"""Summarise an ncu `--page source --csv --print-source sass` export: stall
samples per instruction class and the hottest SASS lines (diagnostics)."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
by_op = defaultdict(lambda: defaultdict(float))
lines = []
for r in data:
    if len(r) < len(hdr):
        continue
    src = r[col["Source"]].strip()
    op = re.sub(r"^@!?U?P\d+\s+", "", src).split(" ")[0]
    samples = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    tot += samples
    by_op[op]["samples"] += samples
    by_op[op]["exec"] += float(r[col["Instructions Executed"]] or 0)
    for s in stall_cols:
        v = float(r[col[s]] or 0)
        by_op[op][s] += v
    lines.append((samples, r[col["Address"]], src, {s: float(r[col[s]] or 0) for s in stall_cols}))
print(f"total samples {tot:.0f}")
print("per opcode (share of samples, executed warp-instr, top stalls):")
for op, d in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:25]:
    st = sorted(((k, v) for k, v in d.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:4]
    print(f"  {op:28s} {100 * d['samples'] / tot:5.1f}%  exec {d['exec']:12.0f}  " +
          " ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in st if v > 0))
agg = defaultdict(float)
for _, _, _, st in lines:
    for k, v in st.items():
        agg[k] += v
print("stall reasons overall:", " ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0))
print("hottest lines:")
for s, a, src, st in sorted(lines, key=lambda x: -x[0])[:30]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"  {100 * s / tot:5.2f}% {a[-5:]} {src[:60]:60s} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in top if v > 0))
