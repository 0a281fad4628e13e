mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_daop.py -q -x -k "skinny or graph or sequence or gemm" > gpurun_out/p_o.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_o.log
timeout 600 python scripts/prefill_breakdown.py 8 > gpurun_out/prefill_breakdown.txt 2>&1; echo "pb rc=$?"; cat gpurun_out/prefill_breakdown.txt
timeout 600 python scripts/daop32.py --ecr 1.0 --prompt 256 --decode 16 --attention --out gpurun_out/daop32_attn_ecr1.json > gpurun_out/daop32_attn.log 2>&1; echo "daop32 attn rc=$?"; grep -E "prefill_ms|decode_tokens_per_s|setup" gpurun_out/daop32_attn_ecr1.json | head
timeout 300 python scripts/batched_decode_probe.py 64 > gpurun_out/b64.txt 2>&1; echo "b64 rc=$?"; tail -3 gpurun_out/b64.txt
