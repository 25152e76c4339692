# round 2: new GPU tests (halo incl. 2-process IPC, P8 through the engines, per-frame gates, f3 vs oracle),
# the full GPU suite, and the TPC tensor-pipe metric of the cuBLAS GEMM from a --set full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_pipeline.py -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -q 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/gemm_full python tools/ncu_calib.py > /dev/null 2>&1
ncu -i gpurun_out/gemm_full.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:]:
    d=dict(zip(h,r))
    for k,v in d.items():
        if 'pipe_tensor' in k or 'gpu__time_duration.sum' in k or 'mem_tensor' in k: print(k, v)
" > gpurun_out/gemm_tpc.txt
cat gpurun_out/gemm_tpc.txt | head
echo done
