cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
echo done
