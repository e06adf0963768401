#!/bin/bash
# Closing measurement r2h1 (scripts/gpu_final.sh) + ncu source-level capture of the C4 reverse launches
cd "$GRAFT_REPO_ROOT" || cd /root/repo
bash scripts/gpu_final.sh r2h1
CMD="python bench.py --config C4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_bwd_kernel' -s 8 -c 4 -o gpurun_out/prof_r3e_C4bwd $CMD > gpurun_out/ncu_r3e_C4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_r3e_C4.log
