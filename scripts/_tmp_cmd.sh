M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"

for G in -2 -4 -8 64; do
echo "== down group $G"
DAOP_GROUP=$G timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm_pair -s 3 -c 1 python scripts/profile_target.py prefill 2>&1 | grep -E "grouped_gemm|duration|tensor|dram__bytes|hit_rate|per_second" | sed 's/(CUtensorMap_st.*//'
done
