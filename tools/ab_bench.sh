# A/B/C bench (GPU box), settings alternated: bash tools/ab_bench.sh tag "w1 w2" "<envA>" "<envB>" ...
o=gpurun_out; tag=$1; W=$2; shift 2
for w in $W; do
 for r in 1 2; do
  for e in "$@"; do
   env $e timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-corpus 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w [$e]', d['value'], d['e2e']['value'])" >> $o/${tag}_bench.log
  done
 done
done
