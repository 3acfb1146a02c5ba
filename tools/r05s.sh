cd $GRAFT_REPO_ROOT
O=gpurun_out/r05s; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "transpose" 2>&1 | tail -2
for v in 0 1; do echo "variant $v"; TSF_TRANSPOSE=$v timeout 300 python tools/bench_layout.py 50 2>&1 | tail -2; done
python tools/bench_layout.py 5 > $O/plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none -k regex:transpose -s 2 -c 1 -o $O/transpose python tools/bench_layout.py 5 > $O/ncu.log 2>&1; echo "ncu rc=$?"
