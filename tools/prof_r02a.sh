mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ih_bins_kernel -c 1 -o gpurun_out/ncu_tmatch_bins python tools/workload_once.py tmatch 1 > gpurun_out/p_tm.log 2>&1; echo tm $?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_match_kernel --launch-skip 2 -c 1 -o gpurun_out/ncu_gen_p1 python tools/workload_once.py gen_p1 1 > gpurun_out/p_g1.log 2>&1; echo g1 $?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_match_kernel --launch-skip 4 -c 1 -o gpurun_out/ncu_gen_bhat python tools/workload_once.py gen_bhat 1 > gpurun_out/p_gb.log 2>&1; echo gb $?
