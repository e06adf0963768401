#!/bin/bash
# small-problem kernel rework (no per-thread pointer tables, one factor phase, fused P + row sums,
# one flattened gradient phase): GPU suite, C0/C1 bench lines, phase profile
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_pytest.log
for c in C0 C1; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 >> gpurun_out/r2r_cfg.jsonl 2>> gpurun_out/r2r.err; done
timeout 200 python scripts/small_profile.py C0 > gpurun_out/r2r_small.json 2>&1
timeout 200 python scripts/small_profile.py C1 >> gpurun_out/r2r_small.json 2>&1
