# Validate the timing die map against the ncu fabric-counter map, then time the
# per-die GEMM schedule (development aid, GPU box)
timeout 600 ncu --metrics lts__t_sectors_srcunit_ltcfabric.sum -k regex:die_pair --csv --log-file gpurun_out/die_pair.csv python scripts/die_pair_probe.py > gpurun_out/die_pair.log 2>&1
timeout 120 python scripts/die_probe.py gpurun_out/die_pair.csv > gpurun_out/die_probe.txt 2>&1
bash scripts/gemm_die_probe.sh
