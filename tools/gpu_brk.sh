cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -2
timeout 300 python tools/conv_breakdown.py 2>&1 | grep -v "^ws T=32 [12]\|^fz[12]"
timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
