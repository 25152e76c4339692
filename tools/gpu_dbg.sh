cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -2
for D in 0 19 51; do
  echo -n "dbg=$D "
  DVC_DEBUG_CONV=$D timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('fps %.1f conv_ms %.2f TF/s %.1f clk %s' % (d['value'], r['conv_ms_per_step'], r['achieved'], d['clocks']['sm_mhz']))"
done
