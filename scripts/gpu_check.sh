#!/bin/bash
# Parity tests + one short bench line (1 GPU).  Usage: gpu_check.sh TAG [pytest -k expr] [bench config]
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-chk}
K=${2:-}
CFG=${3:-C3}
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 1200 python -m pytest tests -m gpu -x -q "${KARG[@]}" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
