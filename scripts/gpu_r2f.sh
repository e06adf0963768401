#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 300 python scripts/bwd1_profile.py C3 296 > gpurun_out/r2f_prof.json 2>&1
timeout 300 python scripts/bwd1_profile.py C3 148 >> gpurun_out/r2f_prof.json 2>&1
