# f1 parity tests (attention / transformer / full U-Net); K="expr" selects tests; BENCH=1 adds tools/bench_f1.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q ${K:+-k "$K"} 2>&1 | tail -25
if [ -n "$BENCH" ]; then timeout 600 python tools/bench_f1.py > gpurun_out/f1_${TAG:-x}.jsonl 2> gpurun_out/f1_${TAG:-x}.err; cat gpurun_out/f1_${TAG:-x}.jsonl; tail -3 gpurun_out/f1_${TAG:-x}.err; fi
