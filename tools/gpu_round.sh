#!/bin/bash
# One parametrised GPU call (replaces the per-experiment round scripts).
#
#   TAG=r07 DO="test smoke bench configs launch full" bash tools/gpu_round.sh
#
# DO selects the steps (in this order when present):
#   test     pytest -m gpu (K filter: PYK="expr")
#   smoke    __graft_entry__.smoke()
#   bench    default bench line (the driver's command), STEPS/WARMUP
#   configs  bench lines for CFGS (default "C3 C5"), no cpu baseline
#   launch   ncu launch list (gpu__time_duration, cold, serialised) of the default bench
#   full     one ncu --set full capture per kernel regex in KREGEX (default attn_)
#   sass     SASS instruction histogram of libtsf.so (no GPU needed)
#   dist     tools/dist_check.py at P in PS (needs gpurun --gpus >= P)
#   scale    weak-scaling bench lines at P in PS
# Every step runs under its own timeout; numbers from runs under ncu are never bench values.
set -u
cd "$(dirname "$0")/.."
TAG=${TAG:-scratch}
O=gpurun_out/$TAG
mkdir -p "$O"
DO=${DO:-"test smoke bench launch"}
has() { [[ " $DO " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$O/smi.txt" 2>&1

if has test; then
  timeout ${TTEST:-1500} python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} -rA > "$O/pytest.log" 2>&1
  echo "pytest rc=$?"; tail -3 "$O/pytest.log"
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1
  echo "smoke rc=$?"; tail -1 "$O/smoke.log"
fi
summ() {  # one-line summary of a bench JSON line
  python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d.get("roofline", {})
    print(f"  {sys.argv[1]}: {d['value']:.4g} tok/s  {d['ms_per_step']:.4f} ms/step  frac {r.get('frac', 0):.3f}  "
          f"stages {r.get('stage_ms_per_step')}  clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
except Exception as e:
    print("  no line:", sys.argv[1], e)
PY
}
if has bench; then
  timeout 600 python bench.py --steps ${STEPS:-2000} --warmup ${WARMUP:-10} > "$O/bench.json" 2> "$O/bench.err"
  echo "bench rc=$?"; summ "$O/bench.json"
fi
if has configs; then
  for c in ${CFGS:-C3 C5}; do
    timeout 600 python bench.py --config $c --steps ${CSTEPS:-50} --warmup 5 --no-cpu-baseline > "$O/bench_$c.json" 2> "$O/bench_$c.err"
    echo "bench $c rc=$?"; summ "$O/bench_$c.json"
  done
fi
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline ${BENCHARGS:-}"
if has launch; then
  $CMD > "$O/plain.log" 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file "$O/launches.csv" $CMD > "$O/ncu_launch.log" 2>&1
  echo "launch list rc=$?"
fi
if has full; then
  $CMD > "$O/plain_full.log" 2>&1
  for k in ${KREGEX:-attn_}; do
    t=$(echo "$k" | tr -c 'a-zA-Z0-9_' '_')
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-4} -c 1 -o "$O/full_$t" $CMD > "$O/ncu_full_$t.log" 2>&1
    echo "full capture $k rc=$?"
  done
fi
if has sass; then
  cuobjdump -sass paper_2604_16590_b200/libtsf.so | grep -oE '^\s+/\*[0-9a-f]+\*/\s+[A-Z][A-Z0-9_.]+' | awk '{print $2}' | sed 's/\..*//' | sort | uniq -c | sort -rn > "$O/sass_hist.txt"
  head -40 "$O/sass_hist.txt"
fi
if has dist; then
  for P in ${PS:-2 4}; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM % 80 + 10))$P tools/dist_check.py ${DISTARGS:-} > "$O/dist_$P.log" 2>&1
    echo "dist P=$P rc=$?"; grep -E "DIST|rank" "$O/dist_$P.log" | tail -$((P + 1))
  done
fi
if has scale; then
  for P in ${PS:-2 4}; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM % 80 + 10))7 bench.py --gpus $P --steps ${STEPS:-500} --warmup 10 > "$O/scale_$P.json" 2> "$O/scale_$P.err"
    echo "scale P=$P rc=$?"; summ "$O/scale_$P.json"
  done
fi
ls "$O"
