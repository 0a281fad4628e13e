timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/p_q.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_q.log
timeout 300 python scripts/prefill256_probe.py 256 > gpurun_out/prefill256.txt 2>&1; echo "rc=$?"; cat gpurun_out/prefill256.txt
timeout 600 python scripts/prefill_breakdown.py 8 > gpurun_out/prefill_breakdown.txt 2>&1; echo "pb rc=$?"; cat gpurun_out/prefill_breakdown.txt
