# Per-die GEMM schedule x rasterisation groups under ncu (time, SM clock,
# fabric and DRAM bytes per launch); development aid, GPU box
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/die_sweep.csv python scripts/gemm_die_probe.py 0 off,auto "64/16/8/32,-16/-8/-4/8" > gpurun_out/die_sweep.log 2>&1; echo "ncu rc=$?"
