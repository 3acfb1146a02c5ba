O=gpurun_out/r2q; mkdir -p $O
python tools/bench_next.py --reps 3 > $O/plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o /tmp/gemm python tools/bench_next.py --reps 3 > $O/ncu_gemm.log 2>&1; echo ncu gemm rc=$?
ncu -i /tmp/gemm.ncu-rep --page raw --csv > $O/gemm_raw.csv 2>&1; ncu -i /tmp/gemm.ncu-rep --page details > $O/gemm_details.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attn_bwd_kernel -s 0 -c 1 -o /tmp/bwd python tools/bench_next.py --reps 3 > $O/ncu_bwd.log 2>&1; echo ncu bwd rc=$?
ncu -i /tmp/bwd.ncu-rep --page raw --csv > $O/bwd_raw.csv 2>&1; ncu -i /tmp/bwd.ncu-rep --page details > $O/bwd_details.txt 2>&1
ls -la $O
