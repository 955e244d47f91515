#!/bin/bash
# Full ncu capture (with source) of one launch of the c2 recurrent-split layer-2 cell kernel,
# the attention kernel and the beam step (GPU box, after a clean run of the same command).
OUT=${1:-gpurun_out}
mkdir -p $OUT
export ONMT_USE_GRAPH=0
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-corpus"
$CMD > $OUT/plain_fused.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on \
    -k regex:'tc_gemm_fused_kernel|attention_cluster' -s 40 -c 2 \
    -o $OUT/fused_full $CMD > $OUT/ncu_fused.log 2>&1
echo profile done
