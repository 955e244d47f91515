#!/bin/bash
# Full ncu capture of one launch of each non-generator decode kernel (GPU box).
OUT=${1:-gpurun_out}
mkdir -p $OUT
export ONMT_USE_GRAPH=0
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/plain_small.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on \
    -k regex:'attention_kernel|beam_select|row_reduce_topk|dec_cell|attn_out|tc_gemm_kernel' -s 200 -c 8 \
    -o $OUT/small_full $CMD > $OUT/ncu_small.log 2>&1
echo profile done
