#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r05z; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"; tail -c 300 $O/bench_default.json
timeout 300 python bench.py --steps 2000 --warmup 10 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e'], d['clocks'], d['gpu_launches'])"
timeout 120 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>&1; tail -c 300 $O/bench_ref.json
