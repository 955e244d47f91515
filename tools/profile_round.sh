#!/bin/bash
# Run on the GPU box (gpurun): launch lists (cold and warm L2) + one full ncu capture of each
# decode-step kernel.  Each ncu command runs only after the same command exited 0 without ncu.
set -u
OUT=${1:-gpurun_out}
TAG=${2:-r01}
mkdir -p $OUT
export ONMT_USE_GRAPH=0      # ncu cannot replay kernel nodes of our graph; same kernels, direct launches
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-corpus"
$CMD > $OUT/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 120 --csv \
    --log-file $OUT/${TAG}_launches_cold.csv $CMD > $OUT/${TAG}_ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 3000 -c 120 --csv \
    --log-file $OUT/${TAG}_launches_warm.csv $CMD > $OUT/${TAG}_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:'gen_step_kernel|tc_gemm_fused_kernel|attention_cluster_kernel|beam_step_kernel' -s 300 -c 5 \
    -o $OUT/${TAG}_full $CMD > $OUT/${TAG}_ncu3.log 2>&1
echo profile done
