#!/bin/bash
# single- vs two-pass reverse: MMA mix microbench, A/B bench lines, ncu full capture of tc_bwd1_kernel
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 120 ./scripts/mma_bench > gpurun_out/r2e_mma.json 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph"
for r in two single two single; do
  timeout 600 $B --reverse $r >> gpurun_out/r2e_ab.jsonl 2>> gpurun_out/r2e_ab.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_bwd1_kernel' -s 3 -c 1 -o gpurun_out/r2e_bwd1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph --reverse single --batch 256 > gpurun_out/r2e_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2e_ncu.log
