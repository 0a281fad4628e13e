# staged epilogue stores: tests + ncu per-launch metrics vs unstaged (mode bit 19)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_attention.py tests/test_gpu_bench_shapes.py -q -x > gpurun_out/epi_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/epi_tests.log
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/epi.csv python scripts/gemm_power_sweep.py 1 up:0:64 up:0:64:2048 down:2:-16 down:2:-16:2048 > gpurun_out/epi_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/gemm_power_sweep.py 20 up:0:64 up:0:64:2048 down:2:-16 down:2:-16:2048 up:0:64 up:0:64:2048 down:2:-16 down:2:-16:2048 > gpurun_out/epi_time.txt 2>&1
