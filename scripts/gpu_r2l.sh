#!/bin/bash
# single-pass reverse diagnosis: MMA shape microbench, per-role wait profile, single vs two pass at C3
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 120 ./scripts/mma_bench > gpurun_out/r2l_mma.json 2>&1
timeout 300 python scripts/bwd1_profile.py C3 296 > gpurun_out/r2l_prof.json 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph"
for r in two single; do timeout 600 $B --reverse $r >> gpurun_out/r2l_ab.jsonl 2>> gpurun_out/r2l_ab.err; done
