#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3"
for r in two single two single; do timeout 300 $B --config C4 --reverse $r >> gpurun_out/r2h.jsonl 2>> gpurun_out/r2h.err; done
timeout 300 $B --config C0 >> gpurun_out/r2h.jsonl 2>> gpurun_out/r2h.err
