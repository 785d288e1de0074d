# Session-3 full GPU pass: tests, smoke, bench (ours + reference arm), launch list. Outputs under gpurun_out/s3h_*
nvidia-smi -L > gpurun_out/s3h_smi.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s3h_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/s3h_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3h_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/s3h_smoke.txt
timeout 900 python bench.py > gpurun_out/s3h_bench.json 2> gpurun_out/s3h_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/s3h_bench_ref.json 2> gpurun_out/s3h_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3h_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-attn --no-layer > gpurun_out/s3h_ncu.log 2>&1
