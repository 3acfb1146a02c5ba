O=gpurun_out/r2m; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_bwd.py > $O/pytest_bwd.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_bwd.log; grep -E "block bwd|temporal bwd \(8, 300|temporal bwd \(3, 130" $O/pytest_bwd.log | head
timeout 600 python tools/bench_next.py --reps 20 > $O/next.jsonl 2> $O/next.err; echo next rc=$?; grep -E "backward" $O/next.jsonl | cut -c1-300
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -4 $O/memcheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_bwd.py -k "shape0 or shape1" > $O/memcheck_bwd.log 2>&1; echo "memcheck bwd rc=$?"; tail -3 $O/memcheck_bwd.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?"; tail -4 $O/synccheck_smoke.log
