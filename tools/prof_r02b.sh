mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor_maps.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_tm.log 2>&1; echo "pytest rc $? $(tail -1 gpurun_out/pytest_tm.log)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_tmatch.csv python tools/workload_once.py tmatch 2 > gpurun_out/wo_tmatch.log 2>&1; echo tml $?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ih_bins_kernel -c 1 -o gpurun_out/ncu_bins3 python tools/workload_once.py tmatch 1 > gpurun_out/p_tm.log 2>&1; echo tm $?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_match_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu_gen_p1 python tools/workload_once.py gen_p1 1 > gpurun_out/p_g1.log 2>&1; echo g1 $?
