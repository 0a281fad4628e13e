mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_shapes.py -q -s > gpurun_out/p_shapes.log 2>&1; echo "shapes rc=$?"; grep -E "agreement|passed|failed" gpurun_out/p_shapes.log | tail -8
timeout 1200 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_bench_shapes.py > gpurun_out/p_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json | head -c 1500
