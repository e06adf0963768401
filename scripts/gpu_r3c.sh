#!/bin/bash
# Round-2 session 5: reverse pass with row weights below 2^-41 of the edge scale flushed (their P~
# is zero in both fp16 parts already) so the zero-tile skip drops them (libtmc.so) vs no flush
# (libtmc_noflush.so, -DTMC_FLUSH_LOG2=-1e30f); GPU suite + parity sweep on the default.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_pytest.log
timeout 900 python scripts/parity_sweep.py 4 > gpurun_out/r3c_parity.jsonl 2>&1
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4" "C2"; do
    for L in libtmc.so libtmc_noflush.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r3c.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'dense': d.get('tc_bwd_kernel_ms_dense_no_zero_skip'), 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r3c_ab.jsonl
    done
  done
done
CMD="python bench.py --config C2 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_bwd_kernel' -s 16 -c 2 -o gpurun_out/prof_r3c_C2bwd $CMD > gpurun_out/ncu_r3c_C2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_r3c_C2.log
