timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r2ah_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ah_test.txt
TF_NVCC_EXTRA=-DTF_ATTN_SPLIT_ROWS=2 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TF_NVCC_EXTRA=-DTF_ATTN_SPLIT_ROWS=2 timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -k "not pair or 0" > gpurun_out/r2ah_test_split2.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ah_test_split2.txt
