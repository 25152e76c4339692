# A/B of two library builds on the same box: the full U-Net's per-family split (bench_f1 F1 line)
cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in A B; do
  DVC_LIB=ab/libdvc_$v.so timeout 300 python -c "
import sys; sys.path.insert(0, 'tools'); import bench_f1 as b, json
d = b.full_unet(3); s = d['profiled_split']
print('$v', round(d['frames_per_s'], 1), {k: round(v['ms'], 2) for k, v in s.items() if k.startswith('tf') or k.startswith('attn')})"
done; done
