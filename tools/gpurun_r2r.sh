TF_NVCC_EXTRA=-DTF_ATTN_TRACE TF_ATTN_PAIR=2 timeout 600 python tools/attn_trace_pair2.py > gpurun_out/r2r_trace_pair2.txt 2>&1
python -c "from paper_2605_02953_b200 import _build; _build.build(force=True)"
TF_ATTN_PAIR=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair2 -s 1 -c 1 -o gpurun_out/r2r_attn_pair2 python tools/attn_probe.py --once > gpurun_out/r2r_ncu.log 2>&1
ncu -i gpurun_out/r2r_attn_pair2.ncu-rep --page source --csv > gpurun_out/r2r_attn_pair2_source.csv 2>/dev/null
