O=gpurun_out/r2j; mkdir -p $O
timeout 600 python -m pytest -q tests/test_gpu_bwd.py > $O/pytest_bwd.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_bwd.log
timeout 600 python tools/bench_next.py --reps 20 > $O/next.jsonl 2> $O/next.err; echo next rc=$?; cat $O/next.jsonl | cut -c1-400; tail -3 $O/next.err
