set -x
nvidia-smi -L > gpurun_out/r1_smi.txt
./tools/nvls_probe.bin > gpurun_out/r1_nvls_probe.txt 2>&1; echo "probe rc=$?" >> gpurun_out/r1_nvls_probe.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r1_gputest.txt 2>&1
timeout 900 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.txt 2>&1
