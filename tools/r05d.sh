cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r05d
VARIANTS="96,1,4,0 96,1,6,0 96,1,8,0 96,1,4,2 96,1,6,2 96,1,8,2 96,1,0,2" STEPS=600 bash tools/variant_sweep.sh
TSF_FLASH_FLAGS=2 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > gpurun_out/r05d/trace_pp.txt 2>&1; head -14 gpurun_out/r05d/trace_pp.txt
TSF_FLASH_FLAGS=2 timeout 90 python tools/gpu_debug.py block 8 1000 4 64 | tail -2
