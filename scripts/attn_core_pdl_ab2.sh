# decoder32 A/B of the attention-core PDL, interleaved
for r in 1 2 3; do for f in 0 1; do DAOP_ATTN_CORE_PDL=$f timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-server --no-daop --no-ep > gpurun_out/bench_acp_${r}_$f.json 2>/dev/null; done; done
