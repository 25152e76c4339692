cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "unshuffle or expansion or u8" 2>&1 | tail -2
timeout 300 python tools/bench_configs.py --only C2 2>&1 | tail -1
timeout 300 python bench.py > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err; tail -c 1800 gpurun_out/bench_r2g.json
timeout 600 python tools/bench_configs.py --only C5 2>&1 | tail -1
echo done
