cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r05a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r05a/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r05a/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r05a/pytest.log
timeout 300 python bench.py --steps 2000 --warmup 10 > gpurun_out/r05a/bench.json 2> gpurun_out/r05a/bench.err; echo "bench rc=$?"; cat gpurun_out/r05a/bench.json | cut -c1-900
for cfg in C3 C5; do timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r05a/bench_$cfg.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/r05a/bench_$cfg.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$cfg',d['value'],d['ms_per_step'],r['achieved'],r['frac'],r['stage_ms_per_step'])"; done
