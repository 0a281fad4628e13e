cd build/old_repo && timeout 300 python scripts/server_debug.py 4096 60 > ../../gpurun_out/server_debug_old.txt 2>&1; echo "old srv rc=$?"; tail -3 ../../gpurun_out/server_debug_old.txt
