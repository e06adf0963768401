#!/bin/bash
# Round-2 session 5: column-tile weight flags recorded by a separate instantiation of the row-owner
# pass (per-thread maximum, one mask bit per tile, published once per unit: libtmc.so) vs recorded
# from per-tile sums with a vote and a store per tile in both passes (libtmc_r6a.so) vs the row flush
# alone (libtmc_r5.so); then the closing measurement of libtmc.so.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4"; do
    for L in libtmc.so libtmc_r5.so libtmc_r6a.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r3g.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'dense': d.get('tc_bwd_kernel_ms_dense_no_zero_skip'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r3g_ab.jsonl
    done
  done
done
bash scripts/gpu_final.sh r2i1
