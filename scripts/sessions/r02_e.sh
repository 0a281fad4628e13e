mkdir -p gpurun_out
timeout 600 python scripts/stream_kernels.py 10 > gpurun_out/stream_kernels.json 2>&1; echo "stream rc=$?"; cat gpurun_out/stream_kernels.json
