cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_unet.py -x -q -k "shift_ratio or streaming" 2>&1 | tail -5
timeout 900 python tools/bench_configs.py > gpurun_out/configs_r1.jsonl 2> gpurun_out/configs_r1.err; tail -c 1500 gpurun_out/configs_r1.jsonl; tail -5 gpurun_out/configs_r1.err
