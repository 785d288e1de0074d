# ncu --set full of the fused MoE dispatch (routing in the launch, and routing given) after session 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dispatch_fused_kernel -c 2 -o gpurun_out/ncu_moe_s3 -f python bench.py --only-moe --steps 1 --warmup 1 > gpurun_out/ncu_moe_s3.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_moe_s3.log
