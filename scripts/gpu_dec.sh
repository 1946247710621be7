timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv3x3|v2p" -s 3 -c 3 -o gpurun_out/dec_full python scripts/profile_frame.py --frames 2 > gpurun_out/ncu_d.log 2>&1
tail -2 gpurun_out/ncu_d.log
