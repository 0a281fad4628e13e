# per-die schedule: bit-identity tests + ncu group sweep (development aid)
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "per_die or die_map or grouped_gemm or fused_down" > gpurun_out/die_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/die_tests.log
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/die_sweep2.csv python scripts/gemm_die_probe.py 0 off,auto "64/64/64,-16/-8/-4" > gpurun_out/die_sweep2.log 2>&1; echo "ncu rc=$?"
