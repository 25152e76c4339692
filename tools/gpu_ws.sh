cd $GRAFT_REPO_ROOT
for E in 1 2; do
  echo "=== engine $E"
  DVC_CONV_ENGINE=$E timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "resblock and not 720p" 2>&1 | tail -8
  DVC_CONV_ENGINE=$E timeout 240 python -m pytest tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -8
  DVC_CONV_ENGINE=$E timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -2 | cut -c1-200
  DVC_CONV_ENGINE=$E timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps',d['value'],'conv TF/s',d['roofline']['achieved'],'frac',d['roofline']['frac'],'share',d['roofline']['conv_share_of_step'])"
done
