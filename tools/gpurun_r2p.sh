TF_ATTN_PAIR=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair2 -s 1 -c 1 -o gpurun_out/r2p_attn_pair2 python tools/attn_probe.py --once > gpurun_out/r2p_ncu.log 2>&1
ncu -i gpurun_out/r2p_attn_pair2.ncu-rep --page source --csv > gpurun_out/r2p_attn_pair2_source.csv 2>/dev/null
ncu -i gpurun_out/r2p_attn_pair2.ncu-rep --page details --csv > gpurun_out/r2p_attn_pair2_details.csv 2>/dev/null
