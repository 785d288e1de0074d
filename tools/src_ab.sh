# same-box A/B of two versions of one source file: bash tools/src_ab.sh <csrc file> <alt copy> <bench args...>
f=$1; alt=$2; shift 2
cp paper_2605_02953_b200/csrc/$f /tmp/_ab_cur
for round in 1 2; do
  for which in cur alt; do
    if [ $which = alt ]; then cp $alt paper_2605_02953_b200/csrc/$f; else cp /tmp/_ab_cur paper_2605_02953_b200/csrc/$f; fi
    python -c "import __graft_entry__ as g; g.build()"
    echo "$which: $(timeout 300 python bench.py "$@" 2>&1 | tail -1 | cut -c 1-400)" >> gpurun_out/src_ab.log
  done
done
cp /tmp/_ab_cur paper_2605_02953_b200/csrc/$f
