# attention core launched programmatically behind the QKV GEMV (K / V loads before griddepcontrol.wait) vs plain
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_daop.py -q -x > gpurun_out/acp_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/acp_tests.log
for f in 0 1 0 1; do echo "core_pdl=$f"; DAOP_ATTN_CORE_PDL=$f timeout 300 python scripts/attn_probe.py 512; DAOP_ATTN_CORE_PDL=$f timeout 300 python scripts/attn_probe.py 2000; done > gpurun_out/acp_ab.txt 2>&1
for f in 0 1; do DAOP_ATTN_CORE_PDL=$f timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-server --no-daop --no-ep > gpurun_out/bench_acp$f.json 2>/dev/null; done
