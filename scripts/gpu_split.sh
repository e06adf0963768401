#!/bin/bash
# A/B of the reverse-pass MMA issue split: libtmc (split) vs libtmc_nosplit, parity first.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/split_pytest.log 2>&1; echo rc=$? >> gpurun_out/split_pytest.log
for c in C3 C4 C2; do
  timeout 300 python scripts/kernel_timing.py $c 128 0:3 > gpurun_out/split_$c.log 2>&1
  TMC_LIB_PATH=paper_1806_08593_b200/libtmc_nosplit.so timeout 300 python scripts/kernel_timing.py $c 128 0:3 > gpurun_out/nosplit_$c.log 2>&1
done
