#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 120 ./scripts/mma_bench > gpurun_out/r2b_mma.json 2>&1
timeout 900 python -m pytest tests/test_gpu_elim.py -x -q > gpurun_out/r2b_elim.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_elim.log
