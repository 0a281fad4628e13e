#!/bin/bash
# One GPU session: smoke, GPU tests, bench, ncu launch list + full captures.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
if [ "$1" == "ncu" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_layer|router|perm_|gather|grouped_gemm|combine|skinny|attn_" -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-ep --no-server --no-daop > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_layer -s 3 -c 1 -o gpurun_out/prof_decode -f python scripts/profile_target.py decode > gpurun_out/ncu_decode.log 2>&1; echo "ncu decode rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 2 -c 2 -o gpurun_out/prof_gemm -f python scripts/profile_target.py prefill > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router|gather_bulk|combine_bulk" -s 3 -c 3 -o gpurun_out/prof_router -f python scripts/profile_target.py prefill > gpurun_out/ncu_router.log 2>&1; echo "ncu router rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_prefill_mma|grouped_gemm" -s 3 -c 3 -o gpurun_out/prof_attn_prefill -f python scripts/profile_target.py attn_prefill > gpurun_out/ncu_attn_prefill.log 2>&1; echo "ncu attn prefill rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny -s 4 -c 2 -o gpurun_out/prof_skinny -f python scripts/batched_decode_probe.py 64 > gpurun_out/ncu_skinny.log 2>&1; echo "ncu skinny rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 9 -c 3 -o gpurun_out/prof_attention -f python scripts/attn_probe.py 1000 > gpurun_out/ncu_attention.log 2>&1; echo "ncu attention rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ep_dispatch|ep_recv|ep_publish" -s 4 -c 3 -o gpurun_out/prof_ep -f python -m pytest tests/test_gpu_ep.py -q -x -k "emulated_ranks_equal_single_gpu and 4" > gpurun_out/ncu_ep.log 2>&1; echo "ncu ep rc=$?"
fi
