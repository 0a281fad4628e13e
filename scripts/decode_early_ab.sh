# early PLAN-mode MoE launches behind the O-proj (non-cooperative by default; DAOP_EARLY_COOP=1
# keeps the cooperative attribute): test + decoder32 A/B + timeline
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_daop.py -q -x > gpurun_out/early_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/early_tests.log
for r in 1 2 3; do for f in 0 1; do DAOP_DECODE_EARLY=$f timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-server --no-daop --no-ep --no-prefill > gpurun_out/bench_early_${r}_$f.json 2>/dev/null; done; done
timeout 600 python scripts/decoder_timeline.py > gpurun_out/dec_tl_early.txt 2>&1
