# C4 full-shard error diagnostics, host-delivery roofline probe, C4 panel raster sweep (one B200).
timeout 900 python scripts/diag_fullsize.py c4 64 > gpurun_out/diag_c4.json 2> gpurun_out/diag_c4.err; tail -2 gpurun_out/diag_c4.err; head -12 gpurun_out/diag_c4.json
nvcc -O3 -std=c++17 -arch=sm_100a -Xcompiler -mavx512f scripts/host_pipe_probe.cu -o /tmp/hpp && timeout 600 /tmp/hpp 2>&1 | tee gpurun_out/host_pipe_probe.txt
free -g; lscpu | grep -i "cache\|numa\|model name"
GROUPS_R="4 16" timeout 1200 bash scripts/panel_group_sweep.sh 2>&1 | tee gpurun_out/panel_group_sweep.txt
