#!/bin/bash
# ncu launch list (per-kernel device time, warm L2) of one call of a workload (GPU box)
W=${1:-c4}
OUT=${2:-gpurun_out}
export ONMT_USE_GRAPH=0
CMD="python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-corpus"
$CMD > $OUT/ll_${W}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 2000 -c 600 --csv \
    --log-file $OUT/ll_${W}.csv $CMD > $OUT/ll_${W}_ncu.log 2>&1
python tools/launches.py $OUT/ll_${W}.csv
