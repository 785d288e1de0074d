timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r2ag_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ag_test.txt
bash tools/attn_ab.sh "" "-DTF_ATTN_SPLIT_ROWS=1" ""
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/attn_probe.py --seconds 3 > gpurun_out/r2ag_attn_sustained.txt 2>&1
