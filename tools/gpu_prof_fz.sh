cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fz -s 0 -c 1 -o gpurun_out/prof_fz_$1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fz_$1.log 2>&1
echo done
