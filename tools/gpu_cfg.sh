cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py > gpurun_out/configs_r1.jsonl 2> gpurun_out/configs_r1.err; cat gpurun_out/configs_r1.jsonl; tail -3 gpurun_out/configs_r1.err
