# GEMM policy / group / die re-sweep without the persisting set-aside (ncu per-launch metrics)
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/resweep.csv python scripts/gemm_power_sweep.py 1 up:0:64 up:1:64 up:2:64 up:6:64 up:0:32 up:0:16 down:2:-16 down:0:-16 down:1:-16 down:3:-16 down:2:-8 down:2:-4 > gpurun_out/resweep.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/resweep_die.csv python scripts/gemm_die_probe.py 0 off,auto > gpurun_out/resweep_die.log 2>&1; echo "ncu die rc=$?"
