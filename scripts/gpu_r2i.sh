#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 120 python scripts/small_profile.py C0 > gpurun_out/r2i.json 2>&1
timeout 120 python scripts/small_profile.py C1 >> gpurun_out/r2i.json 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or C0 or C1 or smoke" > gpurun_out/r2i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.log
