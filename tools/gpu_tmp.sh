cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --gpus 2 --share-device --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err; echo rc=$?
tail -c 1500 gpurun_out/bench_n2_shared.json; tail -5 gpurun_out/bench_n2_shared.err
timeout 600 python bench.py --gpus 4 --share-device --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -c 600; echo
timeout 600 python bench.py --gpus 2 --share-device --scaling weak --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -c 400; echo
echo done
