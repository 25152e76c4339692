nvidia-smi; nproc; python -c "import os;print('affinity',len(os.sched_getaffinity(0)))"; lscpu | head -20
ncu --query-metrics --chip gb100 2>/dev/null | grep -i -E "tensor|tmem|umma|pipe_tc" | head -60 > gpurun_out/ncu_metrics.txt
ncu --query-metrics 2>&1 | head -5 >> gpurun_out/ncu_metrics.txt
python -c "import torch;print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))"
