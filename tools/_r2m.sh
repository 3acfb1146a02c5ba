O=gpurun_out/r2m; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_bwd.py > $O/pytest_bwd.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_bwd.log; grep -E "block bwd|temporal bwd \(8, 300|temporal bwd \(3, 130" $O/pytest_bwd.log | head
timeout 600 python tools/bench_next.py --reps 20 > $O/next.jsonl 2> $O/next.err; echo next rc=$?; grep -E "backward" $O/next.jsonl | cut -c1-300
