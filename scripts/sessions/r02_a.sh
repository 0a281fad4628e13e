mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
lscpu > gpurun_out/lscpu.txt
timeout 1200 python -m pytest tests/test_gpu_bench_shapes.py -q -s -x > gpurun_out/p_shapes.log 2>&1; echo "shapes rc=$?"; tail -5 gpurun_out/p_shapes.log
timeout 900 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_bench_shapes.py > gpurun_out/p_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p_gpu.log
CASES="permute router decode prefill ep attention" timeout 1500 bash scripts/sanitize.sh
