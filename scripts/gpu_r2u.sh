#!/bin/bash
# launch lists of C2 and C4 (share of GPU time per kernel)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for c in C2 C4 C0; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2u_$c.csv $CMD > gpurun_out/ncu_launch_r2u_$c.log 2>&1
done
