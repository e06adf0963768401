#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "single_pass" > gpurun_out/r2c_single.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_single.log
