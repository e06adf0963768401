#!/bin/bash
# ncu full capture of the C4 tensor-core launches (forward and reverse) on the closing build
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --config C4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_(fwd|bwd)_kernel' -s 12 -c 6 -o gpurun_out/prof_r3i_C4 $CMD > gpurun_out/ncu_r3i_C4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_r3i_C4.log
