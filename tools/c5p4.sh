#!/bin/bash
# Multi-GPU bench runs with generous timeouts and wall-clock bookkeeping.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/scale
P=${P:-4}
for cfg in ${CFGS:-C5 C2}; do
  t0=$(date +%s)
  timeout ${TMO:-800} python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
    --master-port 29$((RANDOM%90+10))1 bench.py --gpus $P --config $cfg --steps 4 --warmup 3 --no-cpu-baseline \
    > gpurun_out/scale/${cfg}_$P.json 2> gpurun_out/scale/${cfg}_$P.err
  echo "$cfg P=$P exit $? wall $(( $(date +%s) - t0 )) s"
  tail -c 700 gpurun_out/scale/${cfg}_$P.json; echo; grep -v Warning gpurun_out/scale/${cfg}_$P.err | tail -5
done
