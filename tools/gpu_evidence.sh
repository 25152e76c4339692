# Round-end evidence on one B200 (gpurun): GPU tests, smoke, headline bench, per-conv breakdown, ncu
# launch list (+ DRAM bytes), ncu --set full of the first TMA-engine and fused-engine launches, the
# tensor-pipe calibration against cuBLAS, the secondary configs and the f-row benches.
#   TAG=r2 bash tools/gpu_evidence.sh       then locally: python tools/make_profiles.py r2 r2
cd $GRAFT_REPO_ROOT
TAG=${TAG:-ev}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 400 gpurun_out/bench_$TAG.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_$TAG.json 2>&1
timeout 300 python tools/conv_breakdown.py --json gpurun_out/${TAG}_flops.json > gpurun_out/breakdown_$TAG.txt 2>&1
if [ -f ab/libdvc_exp.so ]; then
  DVC_LIB=ab/libdvc_exp.so DVC_FZ_PROF=1 timeout 200 python tools/conv_breakdown.py 2> gpurun_out/fzprof_$TAG.txt > /dev/null
fi
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_ws -s 0 -c 2 -o gpurun_out/prof_convws_$TAG \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_fz -s 0 -c 2 -o gpurun_out/prof_convfz_$TAG \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
TAG=calib_$TAG bash tools/gpu_calib.sh
timeout 900 python tools/bench_configs.py > gpurun_out/configs_$TAG.jsonl 2>&1
timeout 600 python bench.py --attention --steps 5 --warmup 3 > gpurun_out/bench_attn_$TAG.json 2>&1
timeout 600 python tools/bench_f1.py > gpurun_out/f1_$TAG.jsonl 2>&1
timeout 300 python tools/bench_f2.py > gpurun_out/f2_$TAG.jsonl 2>&1
timeout 300 python tools/conv_breakdown.py --vae --frames 8 > gpurun_out/vae_breakdown_$TAG.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:conv_out --csv --log-file gpurun_out/convout_$TAG.csv python tools/vae_once.py 8 > /dev/null 2>&1
timeout 600 python tools/bench_f3.py > gpurun_out/f3_$TAG.jsonl 2>&1
timeout 300 python tools/bench_fp8.py > gpurun_out/fp8_$TAG.jsonl 2>&1
echo done
