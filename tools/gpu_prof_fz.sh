cd $GRAFT_REPO_ROOT
# ncu --set full captures (with source) of the first N fused conv launches of one bench step
timeout 1200 ncu --set full --import-source on -k regex:conv_fz -s ${2:-0} -c ${3:-2} -o gpurun_out/prof_fz_${1:-x} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
