#!/bin/bash
# forward FMA-pipe share: packed-polynomial variants libtmc_pp{2,3,4}.so (4/16, 6/16, 8/16 of the
# exponentials) vs the release (3/16 scalar): parity on the forward tests, interleaved A/B at C3, C4
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for k in 4; do
  TMC_LIB_PATH=$PWD/paper_1806_08593_b200/libtmc_pp$k.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C3 or C4 or extreme" > gpurun_out/r2p_parity_$k.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_parity_$k.log
done
for r in 1 2; do
  for cfg in "C3 --batch 512" "C4"; do
    for L in libtmc.so libtmc_pp2.so libtmc_pp3.so libtmc_pp4.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph --config $cfg 2>>gpurun_out/r2p.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'fwd': d['kernel_ms_per_step'].get('tc_fwd_kernel'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r2p_ab.jsonl
    done
  done
done
