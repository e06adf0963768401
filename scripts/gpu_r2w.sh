#!/bin/bash
# small-problem kernel: round-robin per-latent loops, fp32 max and width-limited shuffles
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug.py -x -q -k "small or C0 or C1 or debug or S_" > gpurun_out/r2w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_pytest.log
for c in C0 C1; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 >> gpurun_out/r2w_cfg.jsonl 2>> gpurun_out/r2w.err; done
timeout 200 python scripts/small_profile.py C0 > gpurun_out/r2w_small.json 2>&1
