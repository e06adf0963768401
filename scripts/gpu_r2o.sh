#!/bin/bash
# wide-softmax forward variant (libtmc_fwdwide.so): parity on the tensor-core forward tests, then an
# interleaved A/B against the release library at C3 (B = 512) and C4
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TMC_LIB_PATH=$PWD/paper_1806_08593_b200/libtmc_fwdwide.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C3 or C4 or ragged or extreme or unequal or 8192" > gpurun_out/r2o_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_parity.log
for r in 1 2; do
  for cfg in "C3 --batch 512" "C4"; do
    for L in libtmc.so libtmc_fwdwide.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --no-graph --config $cfg 2>>gpurun_out/r2o.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'fwd': d['kernel_ms_per_step'].get('tc_fwd_kernel'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r2o_ab.jsonl
    done
  done
done
