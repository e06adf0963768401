#!/bin/bash
# per-config bench lines (C0-C2, C4), per-role wait profiles (forward + two-pass reverse), ncu full
# capture of the single-pass reverse kernel at C3 (B = 256)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3"
for c in C0 C1 C2 C4; do timeout 300 $B --config $c >> gpurun_out/r2m_cfg.jsonl 2>> gpurun_out/r2m.err; done
timeout 300 python scripts/wait_profile.py C3 296 > gpurun_out/r2m_wait.jsonl 2>&1
timeout 300 python scripts/wait_profile.py C4 256 >> gpurun_out/r2m_wait.jsonl 2>&1
timeout 300 python scripts/wait_profile.py C2 512 >> gpurun_out/r2m_wait.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_bwd1_kernel' -s 3 -c 1 -o gpurun_out/r2m_bwd1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph --reverse single --batch 256 > gpurun_out/r2m_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2m_ncu.log
