# round-end evidence: full GPU suite, smoke, headline bench, f-row benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-final}
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.json
timeout 600 python tools/bench_f1.py > gpurun_out/f1_$TAG.jsonl 2>&1
timeout 300 python tools/bench_f2.py > gpurun_out/f2_$TAG.jsonl 2>&1
timeout 600 python tools/bench_f3.py > gpurun_out/f3_$TAG.jsonl 2>&1
timeout 300 python tools/bench_fp8.py > gpurun_out/fp8_$TAG.jsonl 2>&1
echo done
