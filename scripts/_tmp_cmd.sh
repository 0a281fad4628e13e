M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"
timeout 300 python scripts/probe_perf.py prefill 2>&1 | tail -4
for G in 0 16; do
echo "== group $G"
DAOP_GROUP=$G timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 2 -c 2 python scripts/profile_target.py prefill 2>&1 | grep -E "grouped_gemm|duration|tensor|dram__bytes|hit_rate|per_second" | sed 's/(CUtensorMap_st.*//'
done
timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm|Kernel|sm100|nvjet" -c 4 python scripts/_cub.py 2>&1 | grep -E "^  [a-zA-Z_]|duration|tensor|dram__bytes|hit_rate|per_second" | cut -c1-120
