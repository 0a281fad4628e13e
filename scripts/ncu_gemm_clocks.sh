# Per-launch time, DRAM bytes and the SM clock of the prefill GEMM variants vs
# cuBLAS (power-capped clocks; development aid)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__grid_size,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,smsp__inst_executed_pipe_xu.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"nvjet|gemm" --csv --log-file gpurun_out/gemm_clk.csv \
  python scripts/gemm_power_sweep.py 2 cublas_up:0:0 up:0:64 up:0:64:48 up:0:64:4096 up:0:64:12288 up:0:64:8192 \
  cublas_down:0:0 down:2:-16 down:2:-8:48 down:2:-16:4096 down:2:-16:12288 > gpurun_out/gemm_clk.log 2>&1
echo "ncu rc=$?"
timeout 600 python scripts/gemm_power_sweep.py 20 cublas_up:0:0 up:0:64 up:0:64:48 up:0:64:4096 up:0:64:12288 \
  cublas_down:0:0 down:2:-16 down:2:-8:48 down:2:-16:4096 down:2:-16:12288 > gpurun_out/gemm_time.txt 2>&1
echo "time rc=$?"
