# decoder32 / decode32 A/B of the MoE kernel launched by PDL behind the O projection
for r in 1 2 3; do for f in 0 1; do DAOP_MOE_PDL=$f timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-server --no-daop --no-ep --no-prefill > gpurun_out/bench_mp_${r}_$f.json 2>/dev/null; done; done
DAOP_MOE_PDL=1 timeout 600 python scripts/decoder_timeline.py > gpurun_out/dec_tl_mp.txt 2>&1
