#!/bin/bash
# A/B timing of experiment builds on one GPU: tools/ab_run.sh NAME... (exp_libs/libitq3_NAME.so),
# each timed by tools/chain_decomp.py, in alternating order, ROUNDS (default 2) times.
for r in $(seq ${ROUNDS:-2}); do
  for n in "$@"; do
    ITQ3_LIB=exp_libs/libitq3_$n.so python tools/chain_decomp.py 2>/dev/null | tail -1
  done
done
