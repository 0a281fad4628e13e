mkdir -p gpurun_out
timeout 300 python scripts/server_debug.py 4096 60 > gpurun_out/server_debug.txt 2>&1; echo "srv rc=$?"; cat gpurun_out/server_debug.txt | tail -6
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/p_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p_gpu.log
timeout 600 python scripts/prefill_breakdown.py 8 > gpurun_out/prefill_breakdown.txt 2>&1; echo "pb rc=$?"; cat gpurun_out/prefill_breakdown.txt
timeout 600 python scripts/daop32.py --ecr 1.0 --prompt 256 --decode 16 --attention --out gpurun_out/daop32_attn_ecr1.json > gpurun_out/daop32_attn.log 2>&1; echo "daop32 attn rc=$?"; grep -E "prefill_ms|decode_tokens_per_s|setup" gpurun_out/daop32_attn_ecr1.json | head
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_daop_prefill.csv python scripts/profile_target.py daop_prefill256 > /dev/null 2>&1; echo "ncu rc=$?"
