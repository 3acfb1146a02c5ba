#!/bin/bash
# Bench flash-kernel variants: TSF_SUB (64|128) x TSF_SPLIT (1|2) x TSF_EMU x
# TSF_FLASH_FLAGS (1 one MMA issuer, 2 ping-pong), each with a parity check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/var
# VARIANTS="sub,split,emu,flags ..."
for v in ${VARIANTS:-96,1,4,0 96,1,6,0 96,1,8,0 96,1,6,2 64,1,4,0}; do
  set -- ${v//,/ }
  fl=${4:-2}
  tag="$1_$2_$3_$fl"
  TSF_SUB=$1 TSF_SPLIT=$2 TSF_EMU=$3 TSF_FLASH_FLAGS=$fl timeout 120 python bench.py --config ${CFG:-C2} --steps ${STEPS:-1000} --warmup 10 --no-cpu-baseline > gpurun_out/var/v_$tag.json 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
f = f"gpurun_out/var/v_{tag}.json"
try:
    d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f"sub,split,emu,flags={tag}: {d['value']:.4g} tok/s step {d['ms_per_step']:.4f} ms spatial {r['launch_ms']:.4f} ms "
          f"{r['achieved']:.0f} TF/s frac {r['frac']:.3f} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
except Exception as ex:
    print(f"{tag}: failed", open(f).read()[-600:])
PY
  if [ -n "$CHECK" ]; then
    TSF_SUB=$1 TSF_SPLIT=$2 TSF_EMU=$3 TSF_FLASH_FLAGS=$fl timeout 90 python tools/gpu_debug.py block 8 1000 4 64 | tail -2
    TSF_SUB=$1 TSF_SPLIT=$2 TSF_EMU=$3 TSF_FLASH_FLAGS=$fl timeout 90 python tools/gpu_debug.py spatial 4 1000 4 64 iid | tail -2
  fi
done
