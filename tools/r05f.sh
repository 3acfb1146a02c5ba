cd $GRAFT_REPO_ROOT
O=gpurun_out/r05f; mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for sp in 1 2; do
TSF_SPLIT=$sp $CMD > $O/plain$sp.log 2>&1 && \
TSF_SPLIT=$sp timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_flash -c 1 -o $O/flash_s$sp $CMD > $O/ncu$sp.log 2>&1
echo "ncu $sp rc=$?"; tail -2 $O/ncu$sp.log
done
ls -la $O
