#!/bin/bash
# Bench flash-kernel variants: TSF_SUB (64|128) x TSF_SPLIT (1|2) x TSF_EMU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/var
# VARIANTS="sub,split,emu sub,split,emu ..."
for v in ${VARIANTS:-128,1,0 128,1,4 128,1,6 64,1,4 128,2,4 128,2,6}; do
  set -- ${v//,/ }
  TSF_SUB=$1 TSF_SPLIT=$2 TSF_EMU=$3 timeout 120 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/var/v_$1_$2_$3.json 2>&1
  python - "$1" "$2" "$3" <<'PY'
import json, sys
s, sp, e = sys.argv[1:4]
f = f"gpurun_out/var/v_{s}_{sp}_{e}.json"
try:
    d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f"SUB={s} SPLIT={sp} EMU={e}: {d['value']:.4g} tok/s step {d['ms_per_step']:.4f} ms spatial {r['launch_ms']:.4f} ms "
          f"{r['achieved']:.0f} TF/s frac {r['frac']:.3f} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
except Exception as ex:
    print(f"SUB={s} SPLIT={sp} EMU={e}: failed", open(f).read()[-600:])
PY
done
