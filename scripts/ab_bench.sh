#!/bin/bash
# Interleaved A/B of library builds through bench.py (clock drift under the power cap makes
# sequential runs noisy): bash scripts/ab_bench.sh OUT CFG BATCH ROUNDS libA.so libB.so ...
OUT=$1; CFG=$2; BB=$3; R=$4; shift 4
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for r in $(seq 1 $R); do
  for L in "$@"; do
    TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 600 python bench.py --config $CFG --batch $BB --steps 5 --warmup 3 \
      --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph 2>>gpurun_out/$OUT.err \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/$OUT.jsonl
  done
done
