cd $GRAFT_REPO_ROOT
timeout 300 python tools/host_overhead.py 2>&1 | tail -6
timeout 300 python -m pytest tests/test_gpu_unet.py -q -x 2>&1 | tail -2
for T in 1 4 32; do timeout 300 python tools/step_time.py --frames $T --steps 30 2>&1 | tail -1; done
echo done
