# 512-row single-accumulator pair tile vs 256-row double-buffered pair tile (mode bits 12/13), current defaults
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/twom.csv python scripts/gemm_power_sweep.py 1 up:0:64 up:0:64:16 down:2:-16 down:2:-16:32 > gpurun_out/twom.log 2>&1; echo "ncu rc=$?"
