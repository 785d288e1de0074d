timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r2y_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2y_test.txt
for v in 0 2 0 2; do echo "TF_ATTN_PAIR=$v $(TF_ATTN_PAIR=$v timeout 300 python bench.py --only-attn --steps 3 2>/dev/null | tail -1 | cut -c1-330)" >> gpurun_out/r2y_attn_ab.txt; done
TF_ATTN_PAIR=2 timeout 300 python tools/attn_probe.py --seconds 3 > gpurun_out/r2y_attn_sustained.txt 2>&1
timeout 600 python tools/layer_trace.py > gpurun_out/r2y_layer_trace.json 2>&1
