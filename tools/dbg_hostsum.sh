cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in noop torch gloo; do timeout 120 python tools/dbg_hostsum.py $v > gpurun_out/dbg_hs_$v.log 2>&1; done
