#!/bin/bash
# Launch list + full ncu capture of the top kernels of one bench step (1 GPU).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r1}
CFG=${2:-C3}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_(fwd|bwd)_kernel' -s 8 -c 3 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
