#!/bin/bash
# NVLink evidence for the fused communication tiles, one rank per GPU (torchrun).
#
#   bash tools/nvlink_capture.sh N            # on an N-GPU NVSwitch box
#   bash tools/nvlink_capture.sh 2 --dry-run  # 2 ranks sharing one GPU: checks the recipe
#
# Per launch of our kernels on every rank: duration, NVLink TX/RX user bytes, DRAM bytes.
# SM-driven NVLink traffic shows up on the kernel that issues it:
#   gemm_sm100_kernel<...,EPI=1>  GEMM-RS fused scatter epilogue (P2P stores to the owners)
#   rs_reduce_kernel              unfused RS pull-reduce / owner reduce
#   ar_reduce_kernel/ar_nvls_*    GEMM-AR reduce + broadcast (P2P or NVLS)
#   scatter2_kernel / combine*    MoE dispatch scatter / combine pulls
#   gemm_sm100_kernel<...,1>      ag_moe pull-engine CTAs (bulk copies from peers)
# The AG-GEMM pulls are copy-engine transfers (no kernel): their bytes are the
# nvlrx of the window, cross-checked by bench.py's per-op AG time.
# Application replay: kernels that wait on peers' flags cannot be replayed in
# isolation, so every metric here fits one pass.
set -u
N=${1:-8}
DRY=${2:-}
OUT=gpurun_out/nvlink_n${N}
mkdir -p "$OUT"
METRICS=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
KERNELS='regex:gemm_sm100|rs_reduce|ar_reduce|ar_nvls|scatter|combine|agmoe|barrier'
EXTRA="--no-attn --no-layer"
timeout 1500 ncu --target-processes all --replay-mode application --clock-control none \
  --metrics "$METRICS" -k "$KERNELS" -c 200 --csv --log-file "$OUT/launches.csv" \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --gpus "$N" --steps 2 --warmup 1 --no-cpu-baseline --no-e2e $EXTRA \
  > "$OUT/bench_under_ncu.log" 2>&1
echo "ncu rc=$?" >> "$OUT/bench_under_ncu.log"
python tools/nvlink_summary.py "$OUT" > "$OUT/summary.txt" 2>&1
if [ -n "$DRY" ]; then echo "dry run ($N ranks sharing the visible GPUs): NVLink bytes are expected to be 0" >> "$OUT/summary.txt"; fi
cat "$OUT/summary.txt"
