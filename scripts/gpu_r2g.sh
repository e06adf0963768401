#!/bin/bash
# per-config bench lines (kernel-level, graph timing for the small ones) + single/two-pass A/B at C3
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3"
for c in C0 C1 C2 C4; do timeout 300 $B --config $c >> gpurun_out/r2g_cfg.jsonl 2>> gpurun_out/r2g.err; done
for r in two single; do timeout 600 $B --no-graph --reverse $r --steps 5 >> gpurun_out/r2g_ab.jsonl 2>> gpurun_out/r2g.err; done
