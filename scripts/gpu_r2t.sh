#!/bin/bash
# reverse-pass softmax FMA-pipe share with the packed polynomial (libtmc_bp{1,2}.so: 1/8, 1/4 of the
# exponentials) vs the release; plus the release lib's small-kernel tests (256/512-thread selection)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or C0 or C1" > gpurun_out/r2t_small.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_small.log
TMC_LIB_PATH=$PWD/paper_1806_08593_b200/libtmc_bp2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C3 or C4" > gpurun_out/r2t_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_parity.log
for r in 1 2; do
  for cfg in "C3 --batch 512" "C4"; do
    for L in libtmc.so libtmc_bp1.so libtmc_bp2.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph --config $cfg 2>>gpurun_out/r2t.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'bwd': d['kernel_ms_per_step'].get('tc_bwd_kernel'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r2t_ab.jsonl
    done
  done
done
