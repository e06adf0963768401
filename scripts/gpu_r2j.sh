#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 300 python scripts/wait_profile.py C3 296 > gpurun_out/r2j_wait.json 2>&1
timeout 300 python scripts/wait_profile.py C4 256 >> gpurun_out/r2j_wait.json 2>&1
timeout 300 python scripts/wait_profile.py C2 512 >> gpurun_out/r2j_wait.json 2>&1
timeout 120 python scripts/small_profile.py C0 > gpurun_out/r2j_small.json 2>&1
