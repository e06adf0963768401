#!/bin/bash
# forward: pairwise half-merge barriers with a double-buffered merge slot (libtmc.so) vs the
# all-softmax-warp barriers (libtmc_old.so); graph-replay test
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug.py -x -q -k "graph_replay or C3 or C4 or C2 or debug or tensor_core_forward or extreme" > gpurun_out/r2z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_pytest.log
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4" "C2"; do
    for L in libtmc.so libtmc_old.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r2z.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'fwd': d['kernel_ms_per_step'].get('tc_fwd_kernel'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r2z_ab.jsonl
    done
  done
done
