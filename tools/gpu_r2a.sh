# round 2: new halo tests + full GPU suite, smoke, bench (strong N=1), ncu calibration
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_halo.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -c 2500 gpurun_out/bench_r2a.json
TAG=calib bash tools/gpu_calib.sh
echo done
