timeout 600 python -m pytest tests/test_gpu_dropin.py -x -q -k integration 2>&1 | grep -E "Error|error|assert|Exception|^E " | head -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:token_tc_kernel -s 1 -c 1 \
    -o gpurun_out/q17_token_post python scripts/profile_frame.py --config C5 --frames 1 > gpurun_out/q17_ncu.log 2>&1; tail -1 gpurun_out/q17_ncu.log
