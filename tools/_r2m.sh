O=gpurun_out/r2m; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_bwd.py > $O/pytest_bwd.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_bwd.log; grep -E "block bwd|temporal bwd \(8, 300|temporal bwd \(3, 130" $O/pytest_bwd.log | head
timeout 600 python tools/bench_next.py --reps 20 > $O/next.jsonl 2> $O/next.err; echo next rc=$?; grep -E "backward" $O/next.jsonl | cut -c1-300
timeout 900 python -m pytest -q -x tests/test_gpu_dist_sim.py tests/test_gpu_parity.py -k "block_matches or C2_block_every_row and 0 or sim_block or deterministic or nonfinite or large_config" > $O/pytest_stream.log 2>&1; echo "pytest stream rc=$?"; tail -1 $O/pytest_stream.log
for ns in 2 4; do TSF_STREAM_SLOTS=$ns timeout 120 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/b_slots$ns.json 2>&1; python -c "
import json;d=json.loads(open('$O/b_slots$ns.json').read().strip().splitlines()[-1]);r=d['roofline'];print('slots=$ns', round(d['value']/1e6,2),'Mtok/s temporal',r['stage_ms_per_step']['temporal'])"; done
TSF_STREAM_SLOTS=4 timeout 120 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > $O/b_C3.json 2>&1; python -c "
import json;d=json.loads(open('$O/b_C3.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C3 slots=4', round(d['value']/1e6,3),'Mtok/s temporal',r['stage_ms_per_step']['temporal'])"
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_stream.py > $O/trace_stream4.txt 2>&1; tail -1 $O/trace_stream4.txt
