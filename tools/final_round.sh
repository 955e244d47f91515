#!/bin/bash
# Round-end evidence at HEAD (GPU box): bench lines for c2 (default) and c3 / c4 / c5, the c2
# launch lists (cold / warm) and one full ncu capture of the four decode-step kernels.
set -u
OUT=${1:-gpurun_out}
TAG=${2:-r02r}
mkdir -p $OUT
for w in c3 c4 c5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/${TAG}_bench_$w.json 2> $OUT/${TAG}_bench_$w.err
done
bash tools/profile_round.sh $OUT $TAG
python tools/launches.py $OUT/${TAG}_launches_warm.csv > $OUT/${TAG}_launches_summary.txt
echo "--- cold" >> $OUT/${TAG}_launches_summary.txt
python tools/launches.py $OUT/${TAG}_launches_cold.csv >> $OUT/${TAG}_launches_summary.txt
echo final done
