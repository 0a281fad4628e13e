# (historical: the MW = 2 variant was reverted after this A/B)
# two-weight-tile skinny down GEMM (DAOP_SKINNY_MW2): tests + 256-token prefill A/B + per-op probe
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ep.py tests/test_gpu_bench_shapes.py tests/test_gpu_daop.py -q -x > gpurun_out/mw2_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/mw2_tests.log
for r in 1 2; do for f in 0 1; do echo "DAOP_SKINNY_MW2=$f"; DAOP_SKINNY_MW2=$f timeout 600 python scripts/prefill_breakdown.py 32; done; done > gpurun_out/mw2_pf256.txt 2>&1
for f in 0 1; do echo "DAOP_SKINNY_MW2=$f"; DAOP_SKINNY_MW2=$f timeout 300 python scripts/prefill256_probe.py | tail -2; done > gpurun_out/mw2_ops.txt 2>&1
for f in 0 1; do DAOP_SKINNY_MW2=$f timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-daop --no-server --no-decode32 --no-prefill > gpurun_out/bench_mw2_$f.json 2>/dev/null; done
