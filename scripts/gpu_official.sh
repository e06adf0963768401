#!/bin/bash
# Round measurement: the default bench line, its ncu launch list, and one --set full capture of the
# forward and reverse kernels at full C3 size (1 GPU).  Outputs under gpurun_out/ (summaries go to profiles/).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r1}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph"
$CMD > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_(fwd|bwd)_kernel' -s 28 -c 3 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
