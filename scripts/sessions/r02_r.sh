for nt in 32 64 128; do DAOP_DENSE_NT=$nt timeout 300 python scripts/prefill256_probe.py 256 2>&1 | tail -1 | sed "s/^/nt=$nt /"; done
