# Round-2 full GPU pass: tests, smoke, bench (ours + reference arm). Outputs under gpurun_out/$TAG_*
TAG=${TAG:-r2}
nvidia-smi -L > gpurun_out/${TAG}_smi.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
