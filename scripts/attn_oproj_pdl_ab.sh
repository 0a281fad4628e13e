# O projection launched programmatically behind the attention core (Wo streamed before griddepcontrol.wait) vs plain
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_daop.py -q -x > gpurun_out/aop_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/aop_tests.log
for r in 1 2 3; do for f in 0 1; do DAOP_ATTN_OPROJ_PDL=$f timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-server --no-daop --no-ep > gpurun_out/bench_aop_${r}_$f.json 2>/dev/null; done; done
