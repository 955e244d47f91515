# A/B bench helper (GPU box): tests, then each workload with env settings A and B alternated
# usage: bash tools/ab_run.sh "<envA>" "<envB>" tag [workloads]
o=gpurun_out
A="$1"; B="$2"; tag=$3; W=${4:-"c2 c4 c5 c3"}
timeout 900 python -m pytest tests -m gpu -x -q > $o/${tag}_tests.log 2>&1; echo rc=$? >> $o/${tag}_tests.log
for w in $W; do
 for e in "$A" "$B" "$A" "$B"; do
  env $e timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-corpus 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w [$e]', d['value'], d['e2e']['value'])" >> $o/${tag}_bench.log
 done
done
