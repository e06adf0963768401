#!/bin/bash
# Interleaved A/B of two library builds (clock drift under the power cap makes sequential runs noisy):
# bash scripts/ab_timing.sh libA.so libB.so CFG B ROUNDS
A=$1; B=$2; CFG=${3:-C3}; BB=${4:-128}; R=${5:-3}
for r in $(seq 1 $R); do
  for L in $A $B; do
    TMC_LIB_PATH=$L python scripts/kernel_timing.py $CFG $BB 0:3 | sed "s|^|$(basename $L) |"
  done
done
