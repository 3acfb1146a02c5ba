#!/bin/bash
# Round-5 measurement: full GPU tests, smoke, bench lines (C2 default, C3, C5),
# ncu launch list + one --set full capture per attention kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r05; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 300 python bench.py --steps 2000 --warmup 10 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cut -c1-400 $O/bench.json
for cfg in C3 C5; do timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_$cfg.json 2>&1; python -c "
import json;d=json.loads(open('$O/bench_$cfg.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$cfg',d['value'],d['ms_per_step'],r['achieved'],r['frac'],r['stage_ms_per_step'])"; done
timeout 120 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>&1; tail -c 600 $O/bench_ref.json
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 4 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "full capture rc=$?"
ls -la $O
