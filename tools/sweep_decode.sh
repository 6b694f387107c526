#!/bin/bash
# Sweep the decode kernel's lookahead knobs at the bench shape (CUDA-event timing).
for sa in 2 3 4; do for l2 in 0 2 4 8; do
  echo -n "s_ahead=$sa l2_ahead=$l2 "
  ELATTN_DECODE_S_AHEAD=$sa ELATTN_DECODE_L2_AHEAD=$l2 python tools/time_stages.py --B 320 --reps 10 | tail -1
done; done
