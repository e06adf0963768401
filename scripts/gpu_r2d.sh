#!/bin/bash
# round 2 re-entry check: single-pass reverse parity, full GPU suite, smoke, bench C3
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2d_smi.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "single_pass" > gpurun_out/r2d_single.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_single.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2d_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-traffic > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?" >> gpurun_out/r2d_bench.err
