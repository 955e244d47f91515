# launch lists (ncu) of one workload under two env settings: bash tools/ab_ll.sh "<envA>" "<envB>" [workload]
W=${3:-c2}
mkdir -p gpurun_out/llA gpurun_out/llB
env $1 bash tools/ll_workload.sh $W gpurun_out/llA > gpurun_out/llA/summary.txt 2>&1
env $2 bash tools/ll_workload.sh $W gpurun_out/llB > gpurun_out/llB/summary.txt 2>&1
