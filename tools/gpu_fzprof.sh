cd $GRAFT_REPO_ROOT
for k in "$@"; do
echo "== $k"
env $k DVC_FZ_PROF=1 timeout 120 python tools/conv_breakdown.py 2> gpurun_out/fzprof.txt > /dev/null
tail -20 gpurun_out/fzprof.txt | head -4 | sed 's/fzprof //' | cut -c1-330
done
