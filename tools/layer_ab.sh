# same-box A/B of the layer megakernel: current sources vs .ab/old/{tf_layer.cu,layer.py}
cp paper_2605_02953_b200/csrc/tf_layer.cu /tmp/_cur_tf_layer.cu; cp paper_2605_02953_b200/layer.py /tmp/_cur_layer.py
for round in 1 2; do
  for which in cur old; do
    if [ $which = old ]; then cp .ab/old/tf_layer.cu paper_2605_02953_b200/csrc/tf_layer.cu; cp .ab/old/layer.py paper_2605_02953_b200/layer.py;
    else cp /tmp/_cur_tf_layer.cu paper_2605_02953_b200/csrc/tf_layer.cu; cp /tmp/_cur_layer.py paper_2605_02953_b200/layer.py; fi
    python -c "import __graft_entry__ as g; g.build()"
    echo "$which: $(timeout 300 python bench.py --only-layer --steps 6 --warmup 2 2>&1 | tail -1 | cut -c 180-420)" >> gpurun_out/layer_ab.log
  done
done
cp /tmp/_cur_tf_layer.cu paper_2605_02953_b200/csrc/tf_layer.cu; cp /tmp/_cur_layer.py paper_2605_02953_b200/layer.py
