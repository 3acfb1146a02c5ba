O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest -x -q -rA tests/test_gpu_dist_sim.py tests/test_gpu_parity.py -k "block_matches or C2_block_every_row and 0 or nonfinite or sim or deterministic or host_api or large_config" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for v in 0 1; do TSF_STREAM=$v timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/bench_stream$v.json 2>&1; python -c "
import json;d=json.loads(open('$O/bench_stream$v.json').read().strip().splitlines()[-1]);print('stream=$v', d['value'], d['roofline']['stage_ms_per_step'])"; done
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_stream.py > $O/trace_stream.txt 2>&1; cut -c1-300 $O/trace_stream.txt
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > $O/trace_flash.txt 2>&1; cat $O/trace_flash.txt
