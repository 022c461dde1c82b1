#!/bin/bash
# A/B timing of experiment builds on one GPU: tools/ab_run.sh NAME... (exp_libs/libitq3_NAME.so),
# each timed by tools/chain_decomp.py, in alternating order, ROUNDS (default 2) times.
# NAME=lib:ARGS passes ARGS to chain_decomp.py.
for r in $(seq ${ROUNDS:-2}); do
  for n in "$@"; do
    lib=${n%%:*}; args=""; [ "$lib" != "$n" ] && args=${n#*:}
    echo -n "$n "; ITQ3_LIB=exp_libs/libitq3_$lib.so python tools/chain_decomp.py $args 2>/dev/null | tail -1
  done
done
