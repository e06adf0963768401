#!/bin/bash
# small-problem kernel: round-robin gradient items; 256 vs 512 threads per CTA (interleaved) at C0, C1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or C0 or C1" > gpurun_out/r2s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_pytest.log
TMC_LIB_PATH=$PWD/paper_1806_08593_b200/libtmc_sm512.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or C0 or C1" > gpurun_out/r2s_pytest512.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_pytest512.log
for r in 1 2; do for c in C0 C1; do for L in libtmc.so libtmc_sm512.so; do
  TMC_LIB_PATH=$PWD/paper_1806_08593_b200/$L timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 2>> gpurun_out/r2s.err \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$c', 'lib': '$L', 'us': d['ms_per_step']*1000, 'k_us': d['kernel_ms_per_step']['small_kernel']*1000, 'eager_us': d['ms_per_step_eager']*1000}))" >> gpurun_out/r2s_ab.jsonl
done; done; done
timeout 200 python scripts/small_profile.py C0 > gpurun_out/r2s_small.json 2>&1
timeout 200 python scripts/small_profile.py C1 >> gpurun_out/r2s_small.json 2>&1
