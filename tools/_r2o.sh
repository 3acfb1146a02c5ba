O=gpurun_out/r2o; mkdir -p $O
for args in "8 4096 16 64" "1024 1024 8 64"; do TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py $args > $O/trace_$(echo $args | tr ' ' _).txt 2>&1; echo "== $args"; sed -n 2,3p $O/trace_$(echo $args | tr ' ' _).txt; grep "items in" $O/trace_$(echo $args | tr ' ' _).txt; done
for fl in 0 1; do TSF_BWD_FLAGS=$fl timeout 300 python tools/bench_next.py --reps 10 2>/dev/null | grep spatial_attn_backward | cut -c1-120; done
