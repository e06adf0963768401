#!/bin/bash
# root-edge kernels (UP: CTA-wide root_up_kernel; DOWN: warp-per-row fwd/row): GPU suite, C2/C4/C3 lines
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_pytest.log
for c in C2 C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --no-full-step --no-next2 --no-next3 >> gpurun_out/r2v_cfg.jsonl 2>> gpurun_out/r2v.err; done
