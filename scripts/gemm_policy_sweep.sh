# L2 policy / store-hint sweep of the prefill GEMMs (per-die schedule on, the
# default) under ncu: time, SM clock, DRAM and fabric bytes per launch
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/pol_sweep.csv python scripts/gemm_power_sweep.py 1 up:0:64 up:1:64 up:2:64 up:3:64 up:4:64 up:5:64 up:6:64 up:0:64:64 down:2:-16 down:0:-16 down:1:-16 down:3:-16 down:4:-16 down:5:-16 down:2:-16:64 down:2:-8 > gpurun_out/pol_sweep.log 2>&1; echo "ncu rc=$?"
