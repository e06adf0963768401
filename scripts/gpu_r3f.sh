#!/bin/bash
# Round-2 session 5: column tiles that carry no fp16 weight (recorded by the row-owner pass) are not owned by the column-owner pass (libtmc.so, reading R6) vs the row flush alone (libtmc_r5.so); GPU suite + parity sweep.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_pytest.log
timeout 900 python scripts/parity_sweep.py 4 > gpurun_out/r3f_parity.jsonl 2>&1
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4" "C2"; do
    for L in libtmc.so libtmc_r5.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r3f.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'dense': d.get('tc_bwd_kernel_ms_dense_no_zero_skip'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r3f_ab.jsonl
    done
  done
done
