set -u
for d in wt_79533e4 .; do
  (cd $d; ONMT_USE_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 2000 --csv --log-file /root/repo/gpurun_out/sc_ll_$(basename $(pwd) | tr -d .).csv python bench.py --task score --steps 1 --warmup 3 --no-cpu-baseline --no-corpus > /dev/null 2>&1)
done
