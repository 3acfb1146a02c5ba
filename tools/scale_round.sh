#!/bin/bash
# Weak-scaling bench lines (default config, as the driver runs them) at P = 1, 2, 4
# plus the distributed parity check at P = 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/scale
NG=$(nvidia-smi -L | wc -l)
for P in 1 2 4; do
  [ $P -gt $NG ] && continue
  t0=$(date +%s)
  if [ $P -eq 1 ]; then
    timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scale/C2_$P.json 2> gpurun_out/scale/C2_$P.err
  else
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM%90+10))1 bench.py --gpus $P --steps 50 --warmup 5 \
      > gpurun_out/scale/C2_$P.json 2> gpurun_out/scale/C2_$P.err
  fi
  echo "C2 P=$P exit $? wall $(( $(date +%s) - t0 )) s"
  python - $P <<'PY'
import json, sys
P = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/scale/C2_{P}.json").read().strip().splitlines()[-1])
    print(f"  value {d['value']:.4g} tok/s  ms/step {d['ms_per_step']:.4f}  stages {d['roofline']['stage_ms_per_step']}  a2a {d.get('a2a', {}).get('mode', '-')[:40]}")
except Exception as e:
    print("  no line", e)
PY
done
if [ $NG -ge 4 ]; then
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 \
    tools/dist_check.py 32 4096 16 64 2>&1 | grep -E "DIST|rank" | tail -5
fi
