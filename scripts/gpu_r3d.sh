#!/bin/bash
# Round-2 session 5: every role of the reverse pass loads the next unit's live flags one unit ahead (libtmc.so) vs a dependent global load per unit and per streamed tile (libtmc_noprefetch.so); GPU suite + parity sweep.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_pytest.log
timeout 900 python scripts/parity_sweep.py 4 > gpurun_out/r3d_parity.jsonl 2>&1
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4" "C2"; do
    for L in libtmc.so libtmc_noprefetch.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r3d.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'dense': d.get('tc_bwd_kernel_ms_dense_no_zero_skip'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r3d_ab.jsonl
    done
  done
done
