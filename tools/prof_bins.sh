mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ih_bins_kernel -c 1 -o gpurun_out/ncu_bins2 python tools/workload_once.py tmatch 1 > gpurun_out/p_tm.log 2>&1; echo tm $?
