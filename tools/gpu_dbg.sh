cd $GRAFT_REPO_ROOT
run() { echo -n "$1 "; env $1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('fps %.1f conv_ms %.2f TF/s %.1f clk %s' % (d['value'], r['conv_ms_per_step'], r['achieved'], d['clocks']['sm_mhz']))"; }
run "X=0"
run "DVC_FZ_NB=4"
run "DVC_FZ_NB=6"
run "DVC_FZ_NTF=2"
run "DVC_FZ_NTF=3"
run "DVC_DEBUG_CONV=21"
run "DVC_DEBUG_CONV=21 DVC_FZ_NB=4"
