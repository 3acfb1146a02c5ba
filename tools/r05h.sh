cd $GRAFT_REPO_ROOT
for fl in 4 0; do
echo "flags $fl"
TSF_FLASH_FLAGS=$fl timeout 30 python tools/gpu_debug.py block 8 1000 40 64 | tail -1
TSF_FLASH_FLAGS=$fl timeout 30 python tools/gpu_debug.py spatial 8 1000 40 64 iid | tail -1
done
