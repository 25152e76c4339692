# ncu tensor-pipe calibration: the same metric list on a cuBLAS 8192^3 bf16 GEMM and on every conv launch
# of one headline bench step (--clock-control none, as the bench runs); the per-launch algorithmic FLOPs
# come from the library's own records (tools/conv_breakdown.py --json), merged by tools/calib_table.py.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-calib}
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_gemm.csv python tools/ncu_calib.py > /dev/null 2>&1
timeout 300 python tools/conv_breakdown.py --json gpurun_out/${TAG}_flops.json > gpurun_out/${TAG}_breakdown.txt 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:conv --launch-skip 156 --launch-count 52 --csv --log-file gpurun_out/${TAG}_conv.csv python tools/conv_breakdown.py > /dev/null 2>&1
echo calib done
