cd $GRAFT_REPO_ROOT
for T in 4 8 16; do timeout 300 python tools/step_time.py --frames $T --steps 30 2>&1 | tail -1; done
timeout 300 python tools/conv_breakdown.py --frames 4 2>&1 | head -24
timeout 300 python tools/host_overhead.py 2>&1 | tail -3
echo done
