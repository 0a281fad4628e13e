timeout 300 python scripts/prefill256_probe.py 256 > gpurun_out/prefill256.txt 2>&1; echo "rc=$?"; cat gpurun_out/prefill256.txt
