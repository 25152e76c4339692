# tests + bench + launch list + per-conv breakdown + ncu --set full on the first ws and fz launches
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 2500 gpurun_out/bench_$TAG.json
timeout 300 python tools/conv_breakdown.py > gpurun_out/breakdown_$TAG.txt 2>&1
DVC_FZ_PROF=1 timeout 120 python tools/conv_breakdown.py 2> gpurun_out/fzprof_$TAG.txt > /dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_ws -s 0 -c 2 -o gpurun_out/prof_convws_$TAG python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fz -s 0 -c 2 -o gpurun_out/prof_convfz_$TAG python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fullfz_$TAG.log 2>&1
echo done
