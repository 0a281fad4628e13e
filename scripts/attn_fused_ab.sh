# fused attention core + O-proj (modes 1, 2) vs two launches (0): tests, attention-layer probe, decoder32 bench
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/attn_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/attn_tests.log
for f in 0 1 2 0 1 2; do echo "fused=$f"; DAOP_ATTN_FUSED=$f timeout 300 python scripts/attn_probe.py 512; DAOP_ATTN_FUSED=$f timeout 300 python scripts/attn_probe.py 2000; done > gpurun_out/attn_ab.txt 2>&1
for f in 0 1 2; do DAOP_ATTN_FUSED=$f timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-server --no-daop --no-ep > gpurun_out/bench_attn$f.json 2>/dev/null; done
