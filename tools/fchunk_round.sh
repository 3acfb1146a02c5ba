#!/bin/bash
# Fused-exchange head-chunk pipeline: parity (incl. back-to-back calls) and bench at P = 2, 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fc
for P in 2 4; do
  for FC in 1 2; do
    TSF_FUSED_CHUNKS=$FC timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM%90+10))3 tools/dist_check.py $((8*P)) 4096 16 64 2>&1 | grep -E "DIST|rank 0|Error|error" | tail -3
    echo "  ^ dist_check P=$P chunks=$FC"
  done
  TSF_FUSED_CHUNKS=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM%90+10))3 tools/dist_check.py 1024 256 2 64 2>&1 | grep -E "DIST" | tail -1
  echo "  ^ dist_check flash-temporal P=$P chunks=2"
  for FC in 1 2 4; do
    TSF_FUSED_CHUNKS=$FC timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM%90+10))4 bench.py --gpus $P --steps 200 --warmup 5 --no-cpu-baseline \
      > gpurun_out/fc/C2_${P}_$FC.json 2> gpurun_out/fc/C2_${P}_$FC.err
    python - $P $FC <<'PY'
import json, sys
P, FC = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/fc/C2_{P}_{FC}.json").read().strip().splitlines()[-1])
    print(f"P={P} chunks={FC}: value {d['value']:.4g} tok/s ms/step {d['ms_per_step']:.4f} stages {d['roofline']['stage_ms_per_step']}")
except Exception as e:
    print(f"P={P} chunks={FC}: no line", e, open(f"gpurun_out/fc/C2_{P}_{FC}.err").read()[-800:])
PY
  done
done
