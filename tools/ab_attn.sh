# A/B of two library builds on the same box: the attention kernel at the 720p level-0 shape
cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in A B; do echo "$v $(DVC_LIB=ab/libdvc_$v.so DBGS=0 bash tools/gpu_attn_dbg.sh 2>&1 | grep attn)"; done; done
