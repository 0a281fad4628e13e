mkdir -p gpurun_out
timeout 300 python scripts/server_debug.py 4096 100 > gpurun_out/server_debug.txt 2>&1; echo "srv rc=$?"; tail -2 gpurun_out/server_debug.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/p_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p_gpu.log; grep FAILED gpurun_out/p_gpu.log | head
timeout 600 python scripts/prefill_breakdown.py 8 > gpurun_out/prefill_breakdown.txt 2>&1; echo "pb rc=$?"; cat gpurun_out/prefill_breakdown.txt
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1300 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
CASES="decode" timeout 900 bash scripts/sanitize.sh
