#!/bin/bash
# A/B of one environment switch over the BASELINE configs: tools/ab_env.sh AMG_NO_FORMAT_OVERLAP C3 C4 C5
v=$1; shift
for c in "$@"; do
  echo "== $c default"; python tools/prof_step.py $c --reps 4 2>&1 | tail -3
  echo "== $c $v=1"; env $v=1 python tools/prof_step.py $c --reps 4 2>&1 | tail -3
done
