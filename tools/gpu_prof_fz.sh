cd $GRAFT_REPO_ROOT
# one ncu --set full capture (with source) of the first fused conv launch and of the first L0 ws launch
timeout 900 ncu --set full --import-source on -k regex:conv_fz -s 0 -c 2 -o gpurun_out/prof_fz_${1:-x} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
