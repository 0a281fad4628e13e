for v in v6 v7; do (cd build/$v && timeout 300 python scripts/server_debug.py 4096 60 > ../../gpurun_out/server_debug_$v.txt 2>&1; echo "$v rc=$?"; tail -2 ../../gpurun_out/server_debug_$v.txt); done
