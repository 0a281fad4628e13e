# every decode launch programmatic and non-cooperative (DAOP_MOE_PDL=1) vs cooperative: tests + A/B
DAOP_MOE_PDL=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_daop.py tests/test_gpu_attention.py -q -x > gpurun_out/mp_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/mp_tests.log
for r in 1 2 3; do for f in 0 1; do DAOP_MOE_PDL=$f timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-daop --no-ep --no-prefill > gpurun_out/bench_mp2_${r}_$f.json 2>/dev/null; done; done
