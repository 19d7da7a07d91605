#!/bin/bash
# Round 3c: near-field time with and without the fused correction SpMV (FDA_NEAR_NOCORR=1: measurement only)
for c in 2 4; do
  for m in 0 1; do
    FDA_NEAR_NOCORR=$m timeout 300 python tools/stage_times.py --config $c --reps 20 | sed "s/^/nocorr=$m /"
  done
done
