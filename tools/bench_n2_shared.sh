# functional N=2 bench with both ranks on one GPU (IPC team, torchrun): catches N>1 regressions; numbers are not scaling
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/n2_bench.json 2> gpurun_out/n2_bench.err
echo "rc=$?" >> gpurun_out/n2_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/n2_bench_ref.json 2> gpurun_out/n2_bench_ref.err
echo "rc=$?" >> gpurun_out/n2_bench_ref.err
