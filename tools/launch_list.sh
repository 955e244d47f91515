#!/bin/bash
# ncu launch list (per-kernel device time, warm L2) of a few decode steps (GPU box)
OUT=${1:-gpurun_out}
TAG=${2:-ll}
mkdir -p $OUT
export ONMT_USE_GRAPH=0
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-corpus"
$CMD > $OUT/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 3000 -c 120 --csv \
    --log-file $OUT/${TAG}.csv $CMD > $OUT/${TAG}_ncu.log 2>&1
python tools/launches.py $OUT/${TAG}.csv
