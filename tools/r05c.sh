cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r05c}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "temporal_and_spatial or peaky or block_matches or full_C2 or deterministic or degenerate" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C2',d['value'],d['ms_per_step'],r['achieved'],r['frac'],r['stage_ms_per_step'],d['clocks'])"
for cfg in C3 C5; do timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$cfg.json 2>&1; python -c "
import json;d=json.loads(open('$O/bench_$cfg.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$cfg',d['value'],d['ms_per_step'],r['achieved'],r['frac'],r['stage_ms_per_step'])"; done
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > $O/trace_c2.txt 2>&1; head -14 $O/trace_c2.txt
