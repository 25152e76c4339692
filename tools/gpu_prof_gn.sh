cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
timeout 600 ncu --set full --import-source on -k regex:"gn_" -s 6 -c 3 -o gpurun_out/prof_gn_$TAG python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gn_$TAG.log 2>&1
echo done
