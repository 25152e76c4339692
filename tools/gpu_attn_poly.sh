cd $GRAFT_REPO_ROOT
for pp in ${POLYS:-0 3 5}; do echo "poly=$pp"; DVC_ATTN_POLY=$pp DBGS="${DBGS:-0 2}" bash tools/gpu_attn_dbg.sh 2>&1 | grep -v "^dbg=0$"; done
