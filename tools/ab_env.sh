#!/bin/bash
# A/B timing of one pass kernel under two environment settings:
#   tools/ab_env.sh <kind> <n> <reps> "<envA>" "<envB>"
kind=$1; n=$2; reps=$3
for e in "$4" "$5" "$4" "$5"; do
  env $e python tools/prof_kernel.py $kind $n $reps
done
