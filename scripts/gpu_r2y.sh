#!/bin/bash
# programmatic dependent launch: GPU suite with PDL, then interleaved A/B PDL on/off (libtmc_nopdl.so)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_pytest.log
for r in 1 2; do
  for cfg in "C2" "C4" "C3 --batch 512"; do
    for L in libtmc.so libtmc_nopdl.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r2y.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'eager': d['ms_per_step_eager'], 'graph': d['ms_per_step_cuda_graph'], 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r2y_ab.jsonl
    done
  done
done
