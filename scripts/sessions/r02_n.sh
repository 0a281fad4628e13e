mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or combine" > gpurun_out/p_n.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_n.log
timeout 900 python scripts/gemm_power_sweep.py 10 up:0:64 up:0:64:256 down:2:-16 down:2:-16:256 prefill:0:0 prefill:0:0:256 prefill:0:0 prefill:0:0:256 > gpurun_out/gemm_sweep_epi.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/gemm_sweep_epi.txt
