mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/p_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1200 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python scripts/daop32.py --ecr 1.0 --prompt 256 --decode 16 --attention --out gpurun_out/daop32_attn_ecr1.json > gpurun_out/daop32_attn.log 2>&1; echo "daop32 attn rc=$?"; grep -E "prefill_ms|setup" gpurun_out/daop32_attn_ecr1.json | head
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"router|perm_|gather|combine|grouped_gemm" -c 40 --csv --log-file gpurun_out/launches_prefill.csv python scripts/profile_target.py prefill > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router_mma1|gather_bulk|combine_bulk" -s 3 -c 3 -o gpurun_out/prof_small -f python scripts/profile_target.py prefill > gpurun_out/ncu_small.log 2>&1; echo "ncu small rc=$?"
