#!/bin/bash
# ncu source-level capture of one forward and one reverse tensor-core launch (kernel_timing driver, 1 GPU).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-p}
CMD="python scripts/kernel_timing.py C3 256 0:3:0"
$CMD > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_fwd_kernel' -s 14 -c 1 -o gpurun_out/prof_fwd_$TAG $CMD > gpurun_out/ncu_fwd_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'tc_bwd_kernel' -s 29 -c 2 -o gpurun_out/prof_bwd_$TAG $CMD > gpurun_out/ncu_bwd_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_bwd_$TAG.log
