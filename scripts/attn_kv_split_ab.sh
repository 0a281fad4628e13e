# prompt attention with the KV range split over two warp groups (DAOP_ATTN_KV_SPLIT) vs one
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_daop.py -q -x > gpurun_out/kvs_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/kvs_tests.log
for r in 1 2; do for f in 0 1; do echo "KV_SPLIT=$f"; DAOP_ATTN_KV_SPLIT=$f timeout 300 python scripts/prefill256_probe.py | tail -1; DAOP_ATTN_KV_SPLIT=$f timeout 600 python scripts/prefill_breakdown.py 32 | grep "attention=True: 0"; done; done > gpurun_out/kvs_ab.txt 2>&1
