#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
python scripts/kernel_timing.py C3 128 3:3 > gpurun_out/exp1_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp1_launch_f0.csv python scripts/kernel_timing.py C3 128 0:3 > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp1_launch_f3.csv python scripts/kernel_timing.py C3 128 3:3 > /dev/null 2>&1 &&
TMC_DEBUG_FLAGS=3 ncu --set full --clock-control none --import-source on -k regex:tc_fwd -s 8 -c 1 -o gpurun_out/prof_fwd_skel python scripts/kernel_timing.py C3 128 3:3 > gpurun_out/exp1_ncu.log 2>&1
echo rc=$? >> gpurun_out/exp1_ncu.log
