# (mode bit 23 = SwiGLU epilogue without overlapped TMEM reads)
# overlapped TMEM reads in the up GEMM epilogue vs not (mode bit 23): tests + ncu A/B
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bench_shapes.py tests/test_gpu_ep.py -q -x > gpurun_out/silu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/silu_tests.log
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed_pipe_xu.sum,sm__inst_executed.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/silu.csv python scripts/gemm_power_sweep.py 1 up:0:64 up:0:64:32768 up:0:64 up:0:64:32768 > gpurun_out/silu_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/gemm_power_sweep.py 20 up:0:64 up:0:64:32768 up:0:64 up:0:64:32768 > gpurun_out/silu_time.txt 2>&1
