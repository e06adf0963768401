#!/bin/bash
# Round-2 closing measurement (1 GPU): GPU suite, parity sweep, default bench line (C3, with traffic,
# e2e, cpu baseline, side legs), per-config lines (C0-C2, C4), launch list + full capture of the
# dominant kernels, reference arm.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r2final}
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python scripts/parity_sweep.py 6 > gpurun_out/parity_sweep_$TAG.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3"
for c in C0 C1 C2 C4; do timeout 300 $B --config $c >> gpurun_out/cfg_$TAG.jsonl 2>> gpurun_out/cfg_$TAG.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/reference_$TAG.json 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_(fwd|bwd)_kernel' -s 20 -c 3 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
