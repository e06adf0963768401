#!/bin/bash
# Round-2 session 5: forward softmax with optimistic (no maximum scan) tiles and an exact fallback
# (libtmc_mf.so: -DTMC_FWD_MAXFREE=1; libtmc_mf3.so: + 6/16 of the exponentials on the FMA pipe)
# vs the default; ncu full capture of the C2 kernels (where does the K = 256 reverse pass wait?).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TMC_LIB_PATH=$PWD/paper_1806_08593_b200/libtmc_mf.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r3b_pytest_mf.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_pytest_mf.log
for r in 1 2 3; do
  for cfg in "C3 --batch 512" "C4" "C2"; do
    for L in libtmc.so libtmc_mf.so libtmc_mf3.so; do
      TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 --config $cfg 2>>gpurun_out/r3b.err \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'lib': '$L', 'ms': d['ms_per_step'], 'k': d['kernel_ms_per_step'], 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/r3b_ab.jsonl
    done
  done
done
CMD="python bench.py --config C2 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-full-step --no-next2 --no-next3 --no-graph --no-traffic"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc_(fwd|bwd)_kernel' -s 24 -c 4 -o gpurun_out/prof_r3b_C2 $CMD > gpurun_out/ncu_r3b_C2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_r3b_C2.log
