timeout 300 python scripts/server_debug.py 4096 > gpurun_out/server_debug.txt 2>&1; echo "srv rc=$?"; cat gpurun_out/server_debug.txt
timeout 900 python -m pytest tests -q -m gpu -x -k "decode or ep or server" > gpurun_out/p_dec.log 2>&1; echo "dec tests rc=$?"; tail -5 gpurun_out/p_dec.log
mkdir -p gpurun_out
timeout 900 python scripts/gemm_power_sweep.py 10 up:0:64 up:0:64:64 up:0:32:64 up:0:128:64 down:2:-16 down:2:-16:64 down:2:-8:64 down:2:-32:64 prefill:0:0 prefill:0:0:64 cublas_up:0:0 cublas_down:0:0 > gpurun_out/gemm_sweep_r02.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/gemm_sweep_r02.txt
for cs in 0 64; do
DAOP_GEMM_MODE=$((cs << 8)) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"grouped_gemm" -c 4 --csv --log-file gpurun_out/gemm_dram_cs$cs.csv python scripts/profile_target.py prefill > /dev/null 2>&1; echo "ncu cs=$cs rc=$?"
done
