#!/bin/bash
# Run on the GPU box (gpurun): launch lists (cold and warm L2) + one full capture of the
# generator.  Each ncu command runs only after the same command exited 0 without ncu.
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
export ONMT_USE_GRAPH=0      # ncu cannot replay kernel nodes of our graph; same kernels, direct launches
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 130 --csv \
    --log-file $OUT/launches_cold.csv $CMD > $OUT/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 4000 -c 130 --csv \
    --log-file $OUT/launches_warm.csv $CMD > $OUT/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gen_persistent -s 20 -c 1 \
    -o $OUT/gen_full $CMD > $OUT/ncu3.log 2>&1
echo profile done
