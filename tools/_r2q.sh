O=gpurun_out/r2q; mkdir -p $O
python tools/bench_next.py --reps 3 > $O/plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o $O/gemm python tools/bench_next.py --reps 3 > $O/ncu_gemm.log 2>&1; echo ncu gemm rc=$?
timeout 600 ncu --set full --clock-control none -k regex:attn_bwd_kernel -s 1 -c 1 -o $O/bwd python tools/bench_next.py --reps 3 > $O/ncu_bwd.log 2>&1; echo ncu bwd rc=$?
