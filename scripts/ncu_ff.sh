mkdir -p gpurun_out
python scripts/probe_ff.py 4096 > gpurun_out/probe_ff.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:face_factor -s 1 -c 1 -o gpurun_out/prof_ff python scripts/probe_ff.py 1184 > gpurun_out/ncu_ff.log 2>&1
