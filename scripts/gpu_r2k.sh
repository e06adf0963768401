#!/bin/bash
# Round-2 measurement on the state at session start: GPU suite, default bench line, launch list,
# one --set full capture of the dominant kernel (1 GPU).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r2k}
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rA > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_(fwd|bwd)_kernel' -s 20 -c 3 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
