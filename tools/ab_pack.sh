# A/B: attention call (qkv pack + kernel) vs kernel alone at the 720p level-0 shape
cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in A B; do
  DVC_LIB=ab/libdvc_$v.so timeout 300 python -c "
import sys; sys.path.insert(0, 'tools'); import bench_f1 as b
r = b.attn(10)['rows'][0]; print('$v', 'call', round(r['call_ms'], 3), 'kernel', round(r['kernel_ms'], 3), 'pack+launch', round(r['call_ms'] - r['kernel_ms'], 3))"
done; done
