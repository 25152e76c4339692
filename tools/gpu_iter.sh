# usage: bash tools/gpu_iter.sh TAG   -- quick parity subset, bench, ncu of two conv launches
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 2 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo done
