#!/bin/bash
# Strong scaling of C3 and C5 (fixed problem) at P = 1, 2, 4 with the round-5 kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r05n; mkdir -p $O
for cfg in C3 C5; do for P in 1 2 4; do
  if [ $P -eq 1 ]; then
    timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > $O/${cfg}_$P.json 2> $O/${cfg}_$P.err
  else
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM%90+10))1 bench.py --config $cfg --gpus $P --steps 30 --warmup 5 --no-cpu-baseline \
      > $O/${cfg}_$P.json 2> $O/${cfg}_$P.err
  fi
  python - $O/${cfg}_$P.json $cfg $P <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d['roofline']
    print(f"{sys.argv[2]} P={sys.argv[3]}: {d['value']:.4g} tok/s  ms/step {d['ms_per_step']:.3f}  spatial {r['achieved']:.0f} TF/s  stages {r['stage_ms_per_step']}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "no line", e)
PY
done; done
