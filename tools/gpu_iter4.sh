cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps',d['value'],'e2e',d.get('e2e',{}).get('value'),'conv TF/s',d['roofline']['achieved'],'frac',d['roofline']['frac'])"
timeout 300 python tools/conv_breakdown.py
DVC_FZ_PROF=1 timeout 120 python tools/conv_breakdown.py 2> gpurun_out/fzprof.txt > /dev/null
tail -20 gpurun_out/fzprof.txt | sed 's/fzprof //'
