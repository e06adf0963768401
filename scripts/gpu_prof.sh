#!/bin/bash
# ncu capture of the forward and reverse tensor-core kernels on a reduced-B step (1 GPU).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-p}
CFG=${2:-C3}
B=${3:-64}
CMD="python bench.py --config $CFG --batch $B --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_fwd_kernel' -s 7 -c 2 -o gpurun_out/prof_fwd_$TAG $CMD > gpurun_out/ncu_fwd_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_bwd_kernel' -s 14 -c 2 -o gpurun_out/prof_bwd_$TAG $CMD > gpurun_out/ncu_bwd_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_prep_kernel' -s 7 -c 1 -o gpurun_out/prof_prep_$TAG $CMD > gpurun_out/ncu_prep_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_bwd_$TAG.log
