mkdir -p gpurun_out
timeout 300 python scripts/server_debug.py 4096 40 > gpurun_out/server_debug.txt 2>&1; echo "srv rc=$?"; cat gpurun_out/server_debug.txt | tail -15
timeout 600 python -m pytest tests/test_gpu_daop.py tests/test_gpu_attention.py -q -x -k "graph or dense or prefill_parity or l2_prefetch" > gpurun_out/p_i.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_i.log
timeout 600 python scripts/prefill_breakdown.py 8 > gpurun_out/prefill_breakdown.txt 2>&1; echo "pb rc=$?"; cat gpurun_out/prefill_breakdown.txt
timeout 600 python scripts/daop32.py --ecr 1.0 --prompt 256 --decode 16 --attention --out gpurun_out/daop32_attn_ecr1.json > gpurun_out/daop32_attn.log 2>&1; echo "daop32 attn rc=$?"; grep -E "prefill_ms|decode_tokens_per_s|setup" gpurun_out/daop32_attn_ecr1.json | head
