M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second
timeout 300 python scripts/gemm_die_probe.py 10 > gpurun_out/die_gemm.txt 2>&1; echo "time rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file gpurun_out/die_gemm.csv python scripts/gemm_die_probe.py 0 > gpurun_out/die_gemm_ncu.log 2>&1; echo "ncu rc=$?"
