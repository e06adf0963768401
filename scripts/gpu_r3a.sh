#!/bin/bash
# Round-2 session 5: reverse-pass epilogue with the owner rows loaded before the accumulator waits
# (libtmc.so) vs the per-8-feature dependent loads (libtmc_old.so, -DTMC_EPI_PREFETCH=0) vs the
# 2-term gradient GEMM P_hi (T_hi + T_lo) (libtmc_gt2.so, -DTMC_GRAD_TERMS=2); GPU suite on the default.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_pytest.log
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4" "C2"; do
    for L in libtmc.so libtmc_old.so libtmc_gt2.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r3a.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r3a_ab.jsonl
    done
  done
done
TMC_LIB_PATH=$PWD/paper_1806_08593_b200/libtmc_gt2.so timeout 900 python scripts/parity_sweep.py 3 > gpurun_out/r3a_parity_gt2.jsonl 2>&1
