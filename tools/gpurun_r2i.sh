timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_megakernel.py -q -x > gpurun_out/r2i_layertest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2i_layertest.txt
for v in 0 1 0 1; do
  TF_LAYER_DIE=$v timeout 600 python bench.py --only-layer --steps 10 --warmup 3 > gpurun_out/r2i_layer_die$v.json 2>> gpurun_out/r2i_layer.err
  echo "die=$v $(cat gpurun_out/r2i_layer_die$v.json | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d.get("ms"), d.get("comparator",{}).get("ms"), d.get("comparator",{}).get("speedup"))')" >> gpurun_out/r2i_layer_ab.txt
done
