cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/scale
t0=$(date +%s)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 \
  tools/dist_check.py 1024 1024 8 64 2>&1 | grep -E "DIST|rank|Error|error" | tail -6
echo "dist_check wall $(( $(date +%s) - t0 ))"
P=4 CFGS=C5 TMO=900 bash tools/c5p4.sh
