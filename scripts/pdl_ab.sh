# PDL across the hot-path kernels (DAOP_PDL=1, default) vs plain launches: tests, 256-token
# 32-layer prefill, batched decode and the prefill layer
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pdl_tests.log
for r in 1 2; do for f in 0 1; do echo "DAOP_PDL=$f"; DAOP_PDL=$f timeout 600 python scripts/prefill_breakdown.py 32; done; done > gpurun_out/pdl_pf256.txt 2>&1
for r in 1 2; do for f in 0 1; do DAOP_PDL=$f timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-daop --no-ep --no-server --no-decode32 > gpurun_out/bench_pdl_${r}_$f.json 2>/dev/null; done; done
