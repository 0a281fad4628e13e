# skinny GEMMs launched with / without PDL (DAOP_PDL_SKINNY): batched decode and the 256-token prefill
for r in 1 2 3; do for f in 0 1; do DAOP_PDL_SKINNY=$f timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-daop --no-ep --no-server --no-decode32 --no-prefill > gpurun_out/bench_pks_${r}_$f.json 2>/dev/null; done; done
for r in 1 2; do for f in 0 1; do echo "DAOP_PDL_SKINNY=$f"; DAOP_PDL_SKINNY=$f timeout 600 python scripts/prefill_breakdown.py 32; done; done > gpurun_out/pks_pf256.txt 2>&1
