cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r05b
timeout 60 ./tools/ubench5 > gpurun_out/r05b/ubench5.txt 2>&1
timeout 120 ./tools/ubench6 > gpurun_out/r05b/ubench6.txt 2>&1
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > gpurun_out/r05b/trace_c2.txt 2>&1
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py 8 4096 16 64 spatial > gpurun_out/r05b/trace_c2_sp.txt 2>&1
for f in gpurun_out/r05b/*.txt; do echo "== $f"; cat $f | head -40; done
