mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_run_single.py tests/test_oracle_cpu.py -q -x > gpurun_out/p_attn.log 2>&1; echo "attn rc=$?"; tail -15 gpurun_out/p_attn.log
timeout 300 python scripts/pin_probe.py 16 > gpurun_out/pin_probe.json 2>&1; echo "pin rc=$?"; cat gpurun_out/pin_probe.json | tail -2
timeout 300 python scripts/host_bw.py > gpurun_out/host_bw.txt 2>&1; echo "hostbw rc=$?"; tail -20 gpurun_out/host_bw.txt
timeout 900 python scripts/daop32.py --ecr 0.75 0.5 0.25 --prompt 256 --decode 16 --export-dir gpurun_out/daop32_golden --out gpurun_out/daop32_r02.json > gpurun_out/daop32.log 2>&1; echo "daop32 rc=$?"; tail -3 gpurun_out/daop32.log | cut -c1-600
CASES="attention prefill" timeout 900 bash scripts/sanitize.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ep_dispatch|ep_recv|ep_publish" -c 6 -o gpurun_out/prof_ep_dispatch -f python -m pytest tests/test_gpu_ep.py -q -x -k "emulated_ranks_equal_single_gpu and 4-8" > gpurun_out/ncu_ep.log 2>&1; echo "ncu ep rc=$?"
